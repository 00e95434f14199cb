// tcgen05 (5th-generation tensor core) inner loop for the node-level channel-mixing GEMMs.
//
//   out[r, n] = sum_k A[r, k] * W[n, k]      rows r possibly addressed through [node][9][C]
//
// One CTA owns a 128-row x NT-column output tile whose FP32 accumulator lives in TMEM
// (128 lanes x NT columns).  The FP32 operands are split on the fly into TF32 pairs
// (x = x_hi + x_lo) and each 8-wide K step issues three tcgen05.mma.kind::tf32:
//     D += A_lo*W_hi ;  D += A_hi*W_lo ;  D += A_hi*W_hi         ("3xTF32": FP32-level accuracy)
// Operands are staged in shared memory in the canonical K-major SWIZZLE_128B layout (8-row x
// 128-byte atoms, 16-byte chunks XOR-swizzled by the row index); one K chunk = 32 floats = one
// swizzle row.  Because the split needs registers, the producer is the whole CTA (coalesced
// float4 loads -> cvt.rna.tf32 -> st.shared), made visible to the tensor core's async proxy with
// fence.proxy.async; a single elected thread issues the MMAs and commits them to an mbarrier that
// gates the reuse of the staging buffer.  The next chunk's global loads are issued before that
// wait, so they overlap the MMAs; several CTAs per SM (<= 65 KB shared memory, <= 128 TMEM
// columns each) overlap each other's epilogues.  The epilogue reads the accumulator back with
// tcgen05.ld (32 lanes x 32 bit, 16 columns at a time): thread t of warp w owns output row
// 32*w + t.
#pragma once

#include <stdlib.h>

#include <algorithm>

#include "tn_gemm.cuh"

namespace tc5 {

constexpr int BM = 128;      // UMMA M
constexpr int KC = 32;       // floats per K chunk = one 128-byte swizzle row
constexpr int THREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    for (long spin = 0; !done; ++spin) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (spin > (1L << 28)) __trap();  // never hang the device on a protocol error
    }
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (cute::UMMA::SmemDescriptor layout):
// start address >> 4 in [0,14), LBO >> 4 in [16,30) (unused for swizzled K-major: 1),
// SBO >> 4 in [32,46) = 1024 B between 8-row atoms, version 1 in [46,48), layout type 2 in [61,64).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr)
{
    uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// kind::tf32 instruction descriptor: D = F32 (bit 4), A = B = TF32 (2 at bits 7 and 10),
// both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
__device__ __forceinline__ uint32_t make_idesc(int n)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16])
{
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// byte offset of the 16-byte chunk (row r, chunk j of 8) inside a [rows][128 B] swizzled tile
__device__ __forceinline__ uint32_t swz(int r, int j)
{
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((j ^ (r & 7)) << 4));
}

__device__ __forceinline__ void split_store(char *hi_base, char *lo_base, uint32_t off, float4 v)
{
    uint32_t h[4], l[4];
    tf32_split(v.x, h[0], l[0]);
    tf32_split(v.y, h[1], l[1]);
    tf32_split(v.z, h[2], l[2]);
    tf32_split(v.w, h[3], l[3]);
    *reinterpret_cast<uint4 *>(hi_base + off) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4 *>(lo_base + off) = make_uint4(l[0], l[1], l[2], l[3]);
}

// NT: output columns per CTA (16..128, multiple of 16); TMEM_COLS: power of two >= max(NT, 32)
template <int PRO, int EPI, int NT>
__global__ void __launch_bounds__(THREADS) gemm_nt_tc5_kernel(GemmBatch batch)
{
    // The tensor core adds into a TMEM accumulator with truncation, which shrinks a long chain of
    // K steps by ~1e-6 relative (measured as a systematic energy error).  Each K chunk therefore
    // gets a fresh accumulator (two of them, used alternately) whose 12 MMAs add the small
    // correction terms first, and the chunks are summed in registers by round-to-nearest FADDs
    // while the next chunk's MMAs run.
    constexpr int ACC_COLS = NT <= 32 ? 32 : (NT <= 64 ? 64 : 128);
    constexpr int TMEM_COLS = 2 * ACC_COLS;
    constexpr int A_PASSES = BM / 16;   // 128 threads cover 16 rows x 8 chunks per pass
    constexpr int W_PASSES = NT / 16;
    const GemmArgs &g = batch.g[blockIdx.z];
    const int m0 = blockIdx.x * BM;
    const int n0 = blockIdx.y * NT;
    if (m0 >= g.M || n0 >= g.N) return;

    extern __shared__ char smem_raw[];
    char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps the shared address space
    char *a_hi = smem, *a_lo = smem + BM * 128;
    char *w_hi = smem + 2 * BM * 128, *w_lo = w_hi + NT * 128;
    __shared__ uint64_t mma_bar;
    __shared__ uint32_t tmem_base_s;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        mbar_init(&mma_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tmem_base_s)),
                     "n"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_d = tmem_base_s;
    NNP_PDL_SYNC();   // barrier and tensor-memory set-up above overlap the previous kernel's tail

    // loader mapping: 8 threads per row (one 16-byte chunk each), 16 rows per pass
    const int lrow = tid >> 3, lchunk = tid & 7;
    const float *a_ptr[A_PASSES];
#pragma unroll
    for (int p = 0; p < A_PASSES; ++p) {
        const int r = m0 + p * 16 + lrow;
        a_ptr[p] = r < g.M ? g.A + (size_t)gemm_phys_row(g, r) * g.lda + lchunk * 4 : nullptr;
    }
    const float *w_ptr[W_PASSES];
#pragma unroll
    for (int p = 0; p < W_PASSES; ++p) {
        const int n = n0 + p * 16 + lrow;
        w_ptr[p] = n < g.N ? g.W + (size_t)n * g.K + lchunk * 4 : nullptr;
    }

    const int nchunks = (g.K + KC - 1) / KC;
    float4 ra[A_PASSES], rw[W_PASSES];
    auto load_chunk = [&](int c) {
        const int k0 = c * KC;
        const bool k_ok = k0 + lchunk * 4 < g.K;
#pragma unroll
        for (int p = 0; p < A_PASSES; ++p) {
            ra[p] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (a_ptr[p] && k_ok) ra[p] = __ldg(reinterpret_cast<const float4 *>(a_ptr[p] + k0));
        }
#pragma unroll
        for (int p = 0; p < W_PASSES; ++p) {
            rw[p] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (w_ptr[p] && k_ok) rw[p] = __ldg(reinterpret_cast<const float4 *>(w_ptr[p] + k0));
        }
    };

    const uint32_t idesc = make_idesc(NT);
    const uint64_t da_hi = make_desc(smem_u32(a_hi)), da_lo = make_desc(smem_u32(a_lo));
    const uint64_t dw_hi = make_desc(smem_u32(w_hi)), dw_lo = make_desc(smem_u32(w_lo));

    float acc[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) acc[i] = 0.0f;
    // thread (warp, lane) owns accumulator lane 32*warp + lane = one output row
    auto drain = [&](int buf) {
#pragma unroll
        for (int c0 = 0; c0 < NT; c0 += 16) {
            float v[16];
            tmem_ld16(tmem_d + (uint32_t)(buf * ACC_COLS) + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[c0 + i] += v[i];
        }
    };

    load_chunk(0);
    for (int c = 0; c < nchunks; ++c) {
        if (c > 0) {
            mbar_wait(&mma_bar, (uint32_t)((c - 1) & 1));   // MMAs of chunk c-1 have read the buffers
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
#pragma unroll
        for (int p = 0; p < A_PASSES; ++p) {
            float4 v = ra[p];
            if (PRO == PRO_SILU) {
                v.x = nnp_silu(v.x);
                v.y = nnp_silu(v.y);
                v.z = nnp_silu(v.z);
                v.w = nnp_silu(v.w);
            }
            split_store(a_hi, a_lo, swz(p * 16 + lrow, lchunk), v);
        }
#pragma unroll
        for (int p = 0; p < W_PASSES; ++p) split_store(w_hi, w_lo, swz(p * 16 + lrow, lchunk), rw[p]);
        // generic-proxy writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dst = tmem_d + (uint32_t)((c & 1) * ACC_COLS);
#pragma unroll
            for (int ks = 0; ks < KC / 8; ++ks) {
                const uint64_t adv = (uint64_t)(ks * 32 >> 4);   // 8 tf32 = 32 bytes along K
                umma_tf32(dst, da_lo + adv, dw_hi + adv, idesc, ks != 0);
                umma_tf32(dst, da_hi + adv, dw_lo + adv, idesc, 1);
            }
#pragma unroll
            for (int ks = 0; ks < KC / 8; ++ks) {
                const uint64_t adv = (uint64_t)(ks * 32 >> 4);
                umma_tf32(dst, da_hi + adv, dw_hi + adv, idesc, 1);
            }
            umma_commit(&mma_bar);
        }
        if (c + 1 < nchunks) load_chunk(c + 1);             // overlaps the MMAs just issued
        if (c > 0) drain((c - 1) & 1);                       // chunk c-1 is complete (waited for above)
    }
    mbar_wait(&mma_bar, (uint32_t)((nchunks - 1) & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    drain((nchunks - 1) & 1);

    // epilogue, phase 1: TMEM -> registers -> shared memory.  Thread (warp, lane) owns accumulator
    // lane 32*warp + lane = one output row; the operand buffers are free now and are reused as a
    // [128][NT] staging tile whose 16-byte chunks are XOR-swizzled by the row so that both the
    // row-per-thread writes here and the row-per-warp reads below are conflict-free.
    constexpr int CH = NT / 4;
    float *stage = reinterpret_cast<float *>(smem);
    {
        const int rr = warp * 32 + lane;
#pragma unroll
        for (int c0 = 0; c0 < NT; c0 += 16) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int pos = ((c0 >> 2) + q) ^ (rr & (CH - 1));
                *reinterpret_cast<float4 *>(stage + rr * NT + pos * 4) =
                    make_float4(acc[c0 + 4 * q], acc[c0 + 4 * q + 1], acc[c0 + 4 * q + 2], acc[c0 + 4 * q + 3]);
            }
        }
    }
    __syncthreads();
    // phase 2: one warp per row, one float4 per lane -> coalesced global stores
    constexpr int ROWS_PER_IT = 32 / CH;          // rows a warp covers per iteration (NT < 128)
#pragma unroll 4
    for (int it = warp * ROWS_PER_IT; it < BM; it += 4 * ROWS_PER_IT) {
        const int rr = it + lane / CH;
        const int ch = lane % CH;
        const int pos = ch ^ (rr & (CH - 1));
        const float4 v = *reinterpret_cast<const float4 *>(stage + rr * NT + pos * 4);
        gemm_epilogue4<EPI>(g, m0 + rr, n0 + ch * 4, v);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "n"(TMEM_COLS)
                     : "memory");
    }
}


__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// tcgen05.mma with the A operand in tensor memory
__device__ __forceinline__ void umma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                             uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(tmem_d), "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

struct StreamSchedule {
    int cta_begin[4];   // CTAs [cta_begin[z], cta_begin[z+1]) serve problem z
};

// ------------------------------------------------------------------------------------------
// Streaming kernel for the channel-mixing GEMMs (N = K = 128), mode 5: the one the step uses.
//
//   out^T[n, r] = sum_k W[n, k] * X[r, k]
//
// The mixes are skinny (M = 9 N_atoms rows against a 128 x 128 weight): 217 MB of HBM traffic and
// 29 us of 3xTF32 tensor time each at config C, i.e. bound by how many bytes are kept in flight.
//   * persistent CTAs bound to one component group; its weight is the MMA's A operand and lives
//     in TENSOR MEMORY for the life of the CTA (TF32 hi part in columns [0,128), lo in [128,256);
//     lane = output channel), so all of shared memory is an activation ring;
//   * activation rows are copied global -> shared with cp.async (16 B per request, written
//     straight into the K-major SWIZZLE_128B layout, no register staging) through a 7-stage
//     ring, five 32-column chunks (80 KB) ahead of the tensor core.  The copied FP32 words ARE
//     the "hi" operand (kind::tf32 reads the top 19 bits); the producer only derives
//     lo = x - trunc_tf32(x);
//   * one thread issues the tcgen05.mma triples into one of two TMEM accumulators ([256,384),
//     [384,512)); four epilogue warps drain the other with tcgen05.ld.  Lane = output channel, so
//     the 32 lanes of a warp hold 32 consecutive channels of one row: every store instruction
//     writes one full 128-byte line, no staging tile.
constexpr int ST_STAGES = 7;
constexpr int ST_LAG = 5;                           // chunks in flight behind the newest request
constexpr int ST_PRODUCERS = 256;
constexpr int ST_EPI_WARPS = 8;                     // two per TMEM lane quadrant, 64 tile rows each
constexpr int ST_THREADS = 128 + 32 + ST_PRODUCERS + 128;
constexpr int ST_STAGE_BYTES = 2 * BM * 128;        // raw (= hi) and lo, 128 rows x 128 B each

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}

template <int N_>
__device__ __forceinline__ void cp_async_wait()
{
    asm volatile("cp.async.wait_group %0;" ::"n"(N_) : "memory");
}

template <int PRO, int EPI>
__global__ void __launch_bounds__(ST_THREADS, 1) gemm_stream_kernel(GemmBatch batch, StreamSchedule sched)
{
    constexpr int N = 128, K = 128, NCHUNK = K / KC;
    extern __shared__ char smem_raw[];
    char *ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t full_bar[ST_STAGES], empty_bar[ST_STAGES], tfull_bar[2], tempty_bar[2], w_bar;
    __shared__ uint32_t tmem_base_s;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int z = 0;
    while (z < 2 && (int)blockIdx.x >= sched.cta_begin[z + 1]) ++z;
    const int my = blockIdx.x - sched.cta_begin[z];
    const int stride = sched.cta_begin[z + 1] - sched.cta_begin[z];
    const GemmArgs &g = batch.g[z];
    const int tiles = (g.M + BM - 1) / BM;

    if (tid == 0) {
        for (int s = 0; s < ST_STAGES; ++s) {
            mbar_init(&full_bar[s], ST_PRODUCERS / 32);     // one arrival per producer warp
            mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull_bar[a], 1);
            mbar_init(&tempty_bar[a], ST_EPI_WARPS);        // one arrival per epilogue warp
        }
        mbar_init(&w_bar, 32 * ST_EPI_WARPS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tmem_base_s)),
                     "n"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = tmem_base_s;

    // weights -> tensor memory (once): lane = output channel n, column k (hi) / 128 + k (lo).
    // All eight epilogue warps take part (two per TMEM lane quadrant, half of K each, two 16-column
    // blocks in flight): the staging is a chain of dependent L2 round trips, ~15 us of fixed cost per
    // launch when four warps walked all of K one block at a time.
    if (warp < 4 || warp >= 13) {
        const int quad_w = warp & 3;
        const int n = quad_w * 32 + lane;
        const float *wrow = g.W + (size_t)n * K;
        const uint32_t lane_addr = tmem_base + ((uint32_t)(quad_w * 32) << 16);
        const int kbeg = warp < 4 ? 0 : K / 2;
#pragma unroll 2
        for (int k0 = kbeg; k0 < kbeg + K / 2; k0 += 16) {
            uint32_t hi[16], lo[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 v = __ldg(reinterpret_cast<const float4 *>(wrow + k0 + 4 * q));
                tf32_split(v.x, hi[4 * q], lo[4 * q]);
                tf32_split(v.y, hi[4 * q + 1], lo[4 * q + 1]);
                tf32_split(v.z, hi[4 * q + 2], lo[4 * q + 2]);
                tf32_split(v.w, hi[4 * q + 3], lo[4 * q + 3]);
            }
            tmem_st16(lane_addr + (uint32_t)k0, hi);
            tmem_st16(lane_addr + (uint32_t)(K + k0), lo);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(&w_bar);        // only the MMA thread waits for the weights; loads start at once
    }
    // Everything above reads only the weights, which no kernel of the step writes less than two
    // launches before a GEMM that uses them, so it runs while the previous kernel drains; the
    // activations may only be touched from here on.
    NNP_PDL_SYNC();

    if (warp >= 5 && warp < 13) {
        // ============================================================ producers (256 threads)
        const int ptid = tid - 160;
        constexpr int PIECES = BM * 8 / ST_PRODUCERS;       // 16-byte pieces per thread per chunk (4)
        const int total = ((tiles - my + stride - 1) / stride) * NCHUNK;
        uint32_t off[PIECES];
#pragma unroll
        for (int p = 0; p < PIECES; ++p) {
            const int idx = ptid + p * ST_PRODUCERS;
            off[p] = swz(idx >> 3, idx & 7);
        }
        auto issue = [&](int it) {
            const int s = it % ST_STAGES;
            const uint32_t ph = (uint32_t)((it / ST_STAGES) & 1);
            mbar_wait(&empty_bar[s], ph ^ 1);
            const int tile = my + (it / NCHUNK) * stride;
            const int k0 = (it % NCHUNK) * KC;
            const uint32_t raw = smem_u32(ring + s * ST_STAGE_BYTES);
#pragma unroll
            for (int p = 0; p < PIECES; ++p) {
                const int idx = ptid + p * ST_PRODUCERS;
                const int r = tile * BM + (idx >> 3);
                const bool ok = r < g.M;
                const float *src = g.A + (size_t)gemm_phys_row(g, ok ? r : 0) * g.lda + k0 + (idx & 7) * 4;
                cp_async16(raw + off[p], src, ok ? 16u : 0u);   // rows past the end are zero-filled
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        auto convert = [&](int it) {
            const int s = it % ST_STAGES;
            char *x_hi = ring + s * ST_STAGE_BYTES, *x_lo = x_hi + BM * 128;
#pragma unroll
            for (int p = 0; p < PIECES; ++p) {
                float4 v = *reinterpret_cast<const float4 *>(x_hi + off[p]);
                if (PRO == PRO_SILU) {
                    v.x = nnp_silu(v.x);
                    v.y = nnp_silu(v.y);
                    v.z = nnp_silu(v.z);
                    v.w = nnp_silu(v.w);
                    *reinterpret_cast<float4 *>(x_hi + off[p]) = v;
                }
                uint4 l;
                l.x = __float_as_uint(v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u));
                l.y = __float_as_uint(v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u));
                l.z = __float_as_uint(v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u));
                l.w = __float_as_uint(v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
                *reinterpret_cast<uint4 *>(x_lo + off[p]) = l;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&full_bar[s]);
        };
        for (int it = 0; it < total + ST_LAG; ++it) {
            if (it < total) issue(it);
            else asm volatile("cp.async.commit_group;" ::: "memory");   // keep the group count uniform
            if (it >= ST_LAG) {
                cp_async_wait<ST_LAG>();            // everything but the newest ST_LAG groups has landed
                convert(it - ST_LAG);
            }
        }
    } else if (warp == 4) {
        // ================================================================ MMA issue (1 thread)
        if (lane == 0) {
            const uint32_t idesc = make_idesc(N);
            int it = 0, tcount = 0;
            mbar_wait(&w_bar, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int tile = my; tile < tiles; tile += stride, ++tcount) {
                const int acc = tcount & 1;
                const uint32_t acc_ph = (uint32_t)((tcount >> 1) & 1);
                mbar_wait(&tempty_bar[acc], acc_ph ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t tmem_d = tmem_base + (uint32_t)(2 * K + acc * N);
                for (int c = 0; c < NCHUNK; ++c, ++it) {
                    const int s = it % ST_STAGES;
                    const uint32_t ph = (uint32_t)((it / ST_STAGES) & 1);
                    char *x_hi = ring + s * ST_STAGE_BYTES, *x_lo = x_hi + BM * 128;
                    mbar_wait(&full_bar[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint64_t dx_hi = make_desc(smem_u32(x_hi)), dx_lo = make_desc(smem_u32(x_lo));
#pragma unroll
                    for (int ks = 0; ks < KC / 8; ++ks) {
                        const uint64_t adv = (uint64_t)(ks * 32 >> 4);
                        const uint32_t kcol = (uint32_t)(c * KC + ks * 8);
                        umma_tf32_ta(tmem_d, tmem_base + K + kcol, dx_hi + adv, idesc, (c | ks) != 0);  // W_lo * X_hi
                        umma_tf32_ta(tmem_d, tmem_base + kcol, dx_lo + adv, idesc, 1);                  // W_hi * X_lo
                        umma_tf32_ta(tmem_d, tmem_base + kcol, dx_hi + adv, idesc, 1);                  // W_hi * X_hi
                    }
                    umma_commit(&empty_bar[s]);
                    if (c + 1 == NCHUNK) umma_commit(&tfull_bar[acc]);
                }
            }
        }
        __syncwarp();
    } else {
        // ==================================================================== epilogue (warps 0-3)
        // Four warps, one per scheduler, have nothing to hide latency behind, so the per-element
        // work is a pointer bump: rows of a tile are walked in order and the [node][9][C]
        // addressing (ncomp rows per node, then a skip of 9 - ncomp rows) is kept incrementally.
        const int quad = warp & 3;                          // TMEM lane quadrant this warp may read
        const int hrow = warp < 4 ? 0 : BM / 2;             // first tile row of this warp's half
        const int n = quad * 32 + lane;                     // accumulator lane = output channel
        const int ncomp = g.ncomp;
        const int wrap = ncomp > 0 ? ncomp : 0x7fffffff;
        const int ldo = g.ldo;
        const int skip = ncomp > 0 ? (9 - ncomp) * ldo : 0;
        const float bias = g.bias ? __ldg(g.bias + n) : 0.0f;
        int tcount = 0;
        for (int tile = my; tile < tiles; tile += stride, ++tcount) {
            const int acc = tcount & 1;
            const uint32_t acc_ph = (uint32_t)((tcount >> 1) & 1);
            const int r0 = tile * BM + hrow;
            const int rows = g.M - r0 < BM / 2 ? g.M - r0 : BM / 2;
            int node = node_of(ncomp, r0);
            int comp = ncomp > 0 ? r0 - node * ncomp : 0;
            const size_t prow = ncomp > 0 ? (size_t)node * 9 + g.q0 + comp : (size_t)r0;
            float *po = g.out + prow * ldo + n;             // element (row r0, channel n); ldaux == ldo
            float *po2 = (EPI == EPI_GATE || EPI == EPI_STORE_SILU) ? g.out2 + prow * ldo + n : nullptr;
            const float *pa = (EPI == EPI_ADD || EPI == EPI_MUL_SILU_GRAD) ? g.aux + prow * ldo + n : nullptr;
            const float *pg = EPI == EPI_GATE ? g.aux + (size_t)node * g.ldaux + 3 * n + g.grp : nullptr;
            int off = 0, goff = 0;                          // running element offsets from po / pg
            bool waited = false;
#pragma unroll 1
            for (int c0 = 0; c0 < BM / 2; c0 += 16) {
                if (c0 >= rows) break;
                // addresses of this block's 16 rows, and every global read issued up front
                int o[16];
                float a[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    o[i] = off;
                    a[i] = 0.0f;
                    if (c0 + i < rows) {
                        if (EPI == EPI_ADD || EPI == EPI_MUL_SILU_GRAD) a[i] = pa[off];
                        if (EPI == EPI_GATE) a[i] = __ldg(pg + goff);
                    }
                    off += ldo;
                    if (++comp == wrap) {
                        comp = 0;
                        off += skip;
                        goff += g.ldaux;
                    }
                }
                if (!waited) {
                    mbar_wait(&tfull_bar[acc], acc_ph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    waited = true;
                }
                float v[16];
                tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(2 * K + acc * N + hrow + c0), v);
                // v[i] = out[row c0 + i][channel n]: the warp's 32 lanes cover one 128-byte line per row
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    if (c0 + i < rows) {
                        const float x = v[i] + bias;
                        if (EPI == EPI_STORE) {
                            po[o[i]] = x;
                        } else if (EPI == EPI_STORE_SILU) {
                            po[o[i]] = x;
                            po2[o[i]] = nnp_silu(x);
                        } else if (EPI == EPI_ADD) {
                            po[o[i]] = x + a[i];
                        } else if (EPI == EPI_MUL_SILU_GRAD) {
                            po[o[i]] = x * nnp_silu_grad(a[i]);
                        } else {
                            po2[o[i]] = x;
                            po[o[i]] = x * nnp_silu(a[i]);
                        }
                    }
                }
            }
            if (!waited) mbar_wait(&tfull_bar[acc], acc_ph);
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(512)
                     : "memory");
    }
}

template <int PRO, int EPI>
static int launch_stream(const GemmBatch &b, int count, cudaStream_t stream)
{
    if (count < 1 || count > 3) return -100;
    for (int i = 0; i < count; ++i)
        if (b.g[i].N != 128 || b.g[i].K != 128 || b.g[i].lda % 4 != 0 ||
            ((EPI == EPI_ADD || EPI == EPI_MUL_SILU_GRAD) && b.g[i].ldaux != b.g[i].ldo) ||
            (int64_t)b.g[i].M * 9 * b.g[i].ldo >= (int64_t)1 << 31)
            return -100;
    constexpr int smem = ST_STAGES * ST_STAGE_BYTES + 1024;
    static NnpPerDeviceOnce once;
    if (once.first(nnp_current_device()))
        cudaFuncSetAttribute(gemm_stream_kernel<PRO, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int num_sms = nnp_sm_count();
    int tiles[3] = {0, 0, 0}, total = 0;
    for (int i = 0; i < count; ++i) {
        tiles[i] = (b.g[i].M + BM - 1) / BM;
        total += tiles[i];
    }
    if (total <= 0) return NNP_OK;
    // CTAs per problem in proportion to its tiles (at least one, at most one per tile)
    StreamSchedule sc{};
    int used = 0;
    for (int i = 0; i < count; ++i) {
        int c = (int)(((int64_t)tiles[i] * num_sms) / total);
        c = std::max(1, std::min(c, tiles[i]));
        if (tiles[i] == 0) c = 0;
        sc.cta_begin[i] = used;
        used += c;
    }
    for (int i = count; i < 4; ++i) sc.cta_begin[i] = used;
    t_nnp_pdl_ask = true;      // NNP_PDL=2: only this kernel starts early (its weight staging overlaps the previous kernel's tail)
    nnp_launch((gemm_stream_kernel<PRO, EPI>), NNP_GRID(used), ST_THREADS, smem, stream, b, sc);
    NNP_CHECK_LAUNCH("gemm_stream");
    return NNP_OK;
}

template <int PRO, int EPI, int NT>
static int launch_nt(const GemmBatch &b, int count, int maxM, int maxN, cudaStream_t stream)
{
    const int smem = 2 * BM * 128 + 2 * NT * 128 + 1024;
    static NnpPerDeviceOnce once;
    if (once.first(nnp_current_device()))
        cudaFuncSetAttribute(gemm_nt_tc5_kernel<PRO, EPI, NT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dim3 grid(NNP_GRID((maxM + BM - 1) / BM), (maxN + NT - 1) / NT, count);
    nnp_launch((gemm_nt_tc5_kernel<PRO, EPI, NT>), grid, THREADS, smem, stream, b);
    NNP_CHECK_LAUNCH("gemm_nt_tc5");
    return NNP_OK;
}

template <int PRO, int EPI>
static int launch(const GemmBatch &b, int count, cudaStream_t stream)
{
    int maxM = 0, maxN = 0;
    for (int i = 0; i < count; ++i) {
        maxM = std::max(maxM, b.g[i].M);
        maxN = std::max(maxN, b.g[i].N);
        if (b.g[i].N != b.g[0].N) {
            nnp_set_error("tc5 gemm: batched problems must share N");
            return NNP_ERR_INVALID;
        }
    }
    if (maxM <= 0) return NNP_OK;
    if (maxN % 128 == 0) return launch_nt<PRO, EPI, 128>(b, count, maxM, maxN, stream);
    if (maxN % 64 == 0) return launch_nt<PRO, EPI, 64>(b, count, maxM, maxN, stream);
    if (maxN % 32 == 0) return launch_nt<PRO, EPI, 32>(b, count, maxM, maxN, stream);
    if (maxN % 16 == 0) return launch_nt<PRO, EPI, 16>(b, count, maxM, maxN, stream);
    return -100;   // shape not covered: caller falls back to the mma.sync tile
}

}  // namespace tc5

template <int PRO, int EPI>
static int gemm_launch(const GemmBatch &b, int count, cudaStream_t stream)
{
    int maxM = 0, maxN = 0;
    for (int i = 0; i < count; ++i) {
        maxM = b.g[i].M > maxM ? b.g[i].M : maxM;
        maxN = b.g[i].N > maxN ? b.g[i].N : maxN;
        if (b.g[i].K % 4 != 0 || b.g[i].lda % 4 != 0) {
            nnp_set_error("gemm: K=%d and lda=%d must be multiples of 4", b.g[i].K, b.g[i].lda);
            return NNP_ERR_INVALID;
        }
    }
    if (maxM <= 0) return NNP_OK;
    // a handful of row tiles (single small molecules) is pure launch latency: the mma.sync tile has
    // no TMEM allocation or weight staging to pay for (measured on the 22-atom config)
    // ... and the per-tile tcgen05 kernel walks its K chunks serially (~2.5 us each), which is what
    // a GEMM over N_atoms rows costs up to ~8k atoms; the mma.sync tile is quicker there
    // (measured at 2 489 atoms: 0.15 vs 0.24 ms for the eight dense GEMMs)
    const bool streamable = maxN == 128 && b.g[0].K == 128;
    static const int dense_tiny_m = getenv("NNP_DENSE_TINY_M") ? atoi(getenv("NNP_DENSE_TINY_M")) : 8192;
    const bool tiny = t_nnp_gemm_mode == 5 && (maxM <= 1024 || (!streamable && maxM <= dense_tiny_m));
    if (t_nnp_gemm_mode >= 2 && !tiny) {
        int rc = -100;
        if (t_nnp_gemm_mode == 5) rc = tc5::launch_stream<PRO, EPI>(b, count, stream);
        if (rc == -100) rc = tc5::launch<PRO, EPI>(b, count, stream);
        if (rc != -100) return rc;
    }
    dim3 grid(NNP_GRID((maxM + GEMM_BM - 1) / GEMM_BM), (maxN + GEMM_BN - 1) / GEMM_BN, count);
    if (t_nnp_gemm_mode)
        nnp_launch((gemm_nt_kernel<PRO, EPI, true>), grid, GEMM_THREADS, 0, stream, b);
    else
        nnp_launch((gemm_nt_kernel<PRO, EPI, false>), grid, GEMM_THREADS, 0, stream, b);
    NNP_CHECK_LAUNCH("gemm_nt");
    return NNP_OK;
}
