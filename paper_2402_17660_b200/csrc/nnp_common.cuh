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
