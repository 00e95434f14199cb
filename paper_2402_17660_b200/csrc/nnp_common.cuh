// Shared helpers for the sm_100a kernels behind include/nnp_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/nnp_b200.h"

#define NNP_WARP 32
#define NNP_FULL_MASK 0xffffffffu

void nnp_set_error(const char *fmt, ...);

#define NNP_CHECK_ARG(cond, msg)                        \
    do {                                                \
        if (!(cond)) {                                  \
            nnp_set_error("invalid argument: %s", msg); \
            return NNP_ERR_INVALID;                     \
        }                                               \
    } while (0)

#define NNP_CHECK_LAUNCH(name)                                                  \
    do {                                                                        \
        cudaError_t err__ = cudaGetLastError();                                 \
        if (err__ != cudaSuccess) {                                             \
            nnp_set_error("launch %s failed: %s", name, cudaGetErrorString(err__)); \
            return NNP_ERR_CUDA;                                                \
        }                                                                       \
    } while (0)

// ---- launch accounting and per-kernel timing (test/bench instrumentation)
// (thread-local: a caller's counters and profile session are its own; the library keeps no
//  process-wide mutable state besides the default GEMM engine, which is an atomic)
extern thread_local int g_nnp_launch_count;
// wraps the grid argument of every launch: counts kernels enqueued by this library
#define NNP_GRID(x) (++g_nnp_launch_count, (x))

// ---- programmatic dependent launch (PDL)
// Every kernel of the library starts with NNP_PDL_SYNC(): wait until the grid it depends on has
// completed (and its writes are visible), then allow the NEXT kernel of the stream to be scheduled.
// With the launch attribute below the next kernel's blocks are placed as soon as the last wave of
// this one has started, run whatever precedes their own NNP_PDL_SYNC() (barrier / tensor-memory
// set-up, constant weights), and wait there: the launch latency and the ramp-up of a kernel overlap
// the tail of its predecessor instead of following it (~60 kernel boundaries per step).  Anything read
// before NNP_PDL_SYNC() must have been written at least two kernels earlier (or never in the step).
// MEASURED (profiles/r2_summary.md): the captured step graph of config C replays in 5.01 ms with the
// attribute against 4.50 ms without (the waiting blocks of the next kernel take SM slots from the
// tail of the running one), 0.266 against 0.273 ms on the 22-atom config A.  The attribute is
// therefore only set with NNP_PDL=1 in the environment; without it NNP_PDL_SYNC() is a no-op.
// NNP_PDL=2 sets it for the streaming mix GEMM alone (its weight staging into tensor memory then
// overlaps the previous kernel's tail): 4.380 vs 4.410 ms on config C, no change on A, D and E.
#if defined(__CUDA_ARCH__)
#define NNP_PDL_SYNC()                                            \
    do {                                                          \
        asm volatile("griddepcontrol.wait;" ::: "memory");        \
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    } while (0)
#else
#define NNP_PDL_SYNC() do { } while (0)
#endif

bool nnp_pdl_enabled();
int nnp_pdl_mode();                        // 0 = never, 1 = every launch, 2 = only launches that ask for it
extern thread_local bool t_nnp_pdl_ask;    // set by a launch site (the streaming GEMM) right before nnp_launch

template <typename... KArgs, typename... Args>
static inline cudaError_t nnp_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                     cudaStream_t stream, Args &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    const int mode = nnp_pdl_mode();
    cfg.numAttrs = (mode == 1 || (mode == 2 && t_nnp_pdl_ask)) ? 1 : 0;
    t_nnp_pdl_ask = false;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// When profiling is on (nnp_profile_begin), NNP_PROF scopes record a cudaEvent pair around the
// launches they enclose; nnp_profile_report sums the elapsed time per label.
void nnp_prof_mark(const char *label, cudaStream_t stream, int begin);
struct NnpProfScope {
    const char *label;
    cudaStream_t stream;
    NnpProfScope(const char *l, cudaStream_t s) : label(l), stream(s) { nnp_prof_mark(l, s, 1); }
    ~NnpProfScope() { nnp_prof_mark(label, stream, 0); }
};
#define NNP_PROF(label, stream) NnpProfScope nnp_prof_scope_##__LINE__(label, stream)

// Per-device one-time setup (cudaFuncSetAttribute is per device): `first(dev)` is true exactly
// once per device ordinal for each static instance, from whichever thread gets there first.
#include <atomic>
struct NnpPerDeviceOnce {
    std::atomic<unsigned long long> done[2];
    bool first(int dev)
    {
        if (dev < 0 || dev >= 128) return true;    // unknown ordinal: just redo the setup
        const unsigned long long bit = 1ull << (dev & 63);
        return (done[dev >> 6].fetch_or(bit) & bit) == 0;
    }
};
static inline int nnp_current_device()
{
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}
static inline int nnp_sm_count()
{
    static std::atomic<int> sms[128];
    const int dev = nnp_current_device();
    if (dev < 0 || dev >= 128) return 148;
    int v = sms[dev].load(std::memory_order_relaxed);
    if (v == 0) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
        sms[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

static inline size_t nnp_align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace; with base == nullptr it only measures.
struct NnpArena {
    char *base;
    size_t offset;
    explicit NnpArena(void *p) : base(static_cast<char *>(p)), offset(0) {}
    template <typename T>
    T *take(size_t count)
    {
        size_t start = nnp_align_up(offset);
        offset = start + count * sizeof(T);
        return base ? reinterpret_cast<T *>(base + start) : nullptr;
    }
    size_t bytes() const { return nnp_align_up(offset); }
};

static inline int nnp_blocks(int64_t work, int per_block)
{
    int64_t b = (work + per_block - 1) / per_block;
    return b < 1 ? 1 : static_cast<int>(b);
}

__device__ __forceinline__ int nnp_lane() { return threadIdx.x & 31; }

__device__ __forceinline__ float nnp_warp_sum(float v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(NNP_FULL_MASK, v, o);
    return v;
}

__device__ __forceinline__ double nnp_warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(NNP_FULL_MASK, v, o);
    return v;
}

// exclusive prefix sums of int32 arrays (three small kernels; see scan.cu)
size_t nnp_scan_temp_ints(int64_t n);
int nnp_exclusive_scan_i32(const int32_t *in, int32_t *out, int64_t n, int32_t *temp,
                           cudaStream_t stream);
