// Node-level channel-mixing GEMMs:  out[r, n] = sum_k A[r, k] * W[n, k]   ("NT": both K-contiguous).
//
// These are the only dense contractions of the TensorNet step (the per-node linears of SURVEY.md
// Appendix A: lt0..lt5, the embedding's scalar MLP, the readout).  Rows can be addressed through
// the [node][9][C] tensor layout so that all I rows, all A rows or all S rows of a node tensor form
// one GEMM with one weight matrix.
//
// Two inner loops behind one interface:
//   MMA = true : tensor cores with the 3xTF32 split (a = a_hi + a_lo, both TF32; the product keeps
//                a_lo*b_hi + a_hi*b_lo + a_hi*b_hi in an FP32 accumulator) -> FP32-level accuracy.
//   MMA = false: plain FP32 FFMA, kept as the numerical cross-check of the split.
#pragma once

#include "nnp_common.cuh"
#include "tn_math.cuh"

enum { PRO_NONE = 0, PRO_SILU = 1 };
enum { EPI_STORE = 0, EPI_MUL_SILU_GRAD = 1, EPI_GATE = 2, EPI_ADD = 3, EPI_STORE_SILU = 4 };
// EPI_STORE_SILU: out = v (kept for the reverse sweep) and out2 = silu(v) (the next linear's input), so
// that the activation is evaluated once per element instead of once per column tile of the consumer

struct GemmArgs {
    const float *A;
    const float *W;
    const float *bias;
    float *out;
    float *out2;
    const float *aux;
    int M, N, K;
    int lda, ldo, ldaux;
    int ncomp, q0, grp;  // ncomp > 0: logical row r -> physical row (r / ncomp) * 9 + q0 + r % ncomp
};

struct GemmBatch {
    GemmArgs g[3];
};

constexpr int GEMM_BM = 64, GEMM_BN = 64, GEMM_BK = 32, GEMM_LD = GEMM_BK + 4, GEMM_THREADS = 256;

// logical row -> physical row of the [node][9][C] layout; the component counts are 1, 3 or 5, so the
// division is by a compile-time constant in every real case (a runtime divide costs ~25 dependent
// instructions and sat on the critical path of the store loop)
__device__ __forceinline__ int phys_row_of(int ncomp, int q0, int r)
{
    switch (ncomp) {
    case 0: return r;
    case 1: return r * 9 + q0;
    case 3: { const int n = r / 3; return n * 9 + q0 + (r - n * 3); }
    case 5: { const int n = r / 5; return n * 9 + q0 + (r - n * 5); }
    default: { const int n = r / ncomp; return n * 9 + q0 + (r - n * ncomp); }
    }
}

__device__ __forceinline__ int node_of(int ncomp, int r)
{
    switch (ncomp) {
    case 0: case 1: return r;
    case 3: return r / 3;
    case 5: return r / 5;
    default: return r / ncomp;
    }
}

__device__ __forceinline__ int gemm_phys_row(const GemmArgs &g, int r) { return phys_row_of(g.ncomp, g.q0, r); }

// x = hi + lo with hi a TF32 value (10-bit mantissa, round to nearest by integer add-and-mask) and
// lo the exact FP32 remainder (the tensor core reads its top 19 bits).  Three integer/FP
// instructions; cvt.rna.tf32.f32 is not used because ptxas expands it into a long NaN/Inf-safe
// sequence on sm_100a, which made the split -- not the MMAs -- the bottleneck of the GEMMs.
__device__ __forceinline__ void tf32_split(float x, uint32_t &hi, uint32_t &lo)
{
    hi = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2])
{
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int EPI>
__device__ __forceinline__ void gemm_epilogue(const GemmArgs &g, int r, int c, float v)
{
    if (r >= g.M || c >= g.N) return;
    const int pr = gemm_phys_row(g, r);
    if (g.bias) v += g.bias[c];
    const size_t o = (size_t)pr * g.ldo + c;
    if (EPI == EPI_STORE) {
        g.out[o] = v;
    } else if (EPI == EPI_STORE_SILU) {
        g.out[o] = v;
        g.out2[o] = nnp_silu(v);
    } else if (EPI == EPI_MUL_SILU_GRAD) {
        g.out[o] = v * nnp_silu_grad(g.aux[(size_t)pr * g.ldaux + c]);
    } else if (EPI == EPI_GATE) {
        const int node = node_of(g.ncomp, r);
        g.out2[o] = v;
        g.out[o] = v * nnp_silu(g.aux[(size_t)node * g.ldaux + 3 * c + g.grp]);
    } else {
        g.out[o] = v + g.aux[(size_t)pr * g.ldaux + c];
    }
}

// four consecutive columns c..c+3 of one row (c % 4 == 0; all leading dimensions % 4 == 0)
template <int EPI>
__device__ __forceinline__ void gemm_epilogue4(const GemmArgs &g, int r, int c, float4 v)
{
    if (r >= g.M || c >= g.N) return;
    const int pr = gemm_phys_row(g, r);
    if (g.bias) {
        const float4 b = __ldg(reinterpret_cast<const float4 *>(g.bias + c));
        v.x += b.x;
        v.y += b.y;
        v.z += b.z;
        v.w += b.w;
    }
    const size_t o = (size_t)pr * g.ldo + c;
    if (EPI == EPI_STORE) {
        *reinterpret_cast<float4 *>(g.out + o) = v;
    } else if (EPI == EPI_STORE_SILU) {
        *reinterpret_cast<float4 *>(g.out + o) = v;
        *reinterpret_cast<float4 *>(g.out2 + o) = make_float4(nnp_silu(v.x), nnp_silu(v.y), nnp_silu(v.z), nnp_silu(v.w));
    } else if (EPI == EPI_MUL_SILU_GRAD) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(g.aux + (size_t)pr * g.ldaux + c));
        v.x *= nnp_silu_grad(a.x);
        v.y *= nnp_silu_grad(a.y);
        v.z *= nnp_silu_grad(a.z);
        v.w *= nnp_silu_grad(a.w);
        *reinterpret_cast<float4 *>(g.out + o) = v;
    } else if (EPI == EPI_GATE) {
        const int node = node_of(g.ncomp, r);
        const float *a = g.aux + (size_t)node * g.ldaux + 3 * c + g.grp;
        *reinterpret_cast<float4 *>(g.out2 + o) = v;
        v.x *= nnp_silu(__ldg(a));
        v.y *= nnp_silu(__ldg(a + 3));
        v.z *= nnp_silu(__ldg(a + 6));
        v.w *= nnp_silu(__ldg(a + 9));
        *reinterpret_cast<float4 *>(g.out + o) = v;
    } else {
        const float4 a = *reinterpret_cast<const float4 *>(g.aux + (size_t)pr * g.ldaux + c);
        v.x += a.x;
        v.y += a.y;
        v.z += a.z;
        v.w += a.w;
        *reinterpret_cast<float4 *>(g.out + o) = v;
    }
}

template <int PRO, int EPI, bool MMA>
__global__ void __launch_bounds__(GEMM_THREADS) gemm_nt_kernel(GemmBatch batch)
{
    NNP_PDL_SYNC();
    const GemmArgs &g = batch.g[blockIdx.z];
    const int m0 = blockIdx.x * GEMM_BM;
    const int n0 = blockIdx.y * GEMM_BN;
    if (m0 >= g.M || n0 >= g.N) return;

    __shared__ __align__(16) float As[GEMM_BM][GEMM_LD];
    __shared__ __align__(16) float Ws[GEMM_BN][GEMM_LD];

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    // tile loaders: 2 float4 per thread for each operand
    int a_row[2], a_k4[2];
    const float *a_ptr[2];
    const float *w_ptr[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int idx = tid + i * GEMM_THREADS;
        a_row[i] = idx >> 3;
        a_k4[i] = (idx & 7) * 4;
        const int r = m0 + a_row[i];
        a_ptr[i] = r < g.M ? g.A + (size_t)gemm_phys_row(g, r) * g.lda + a_k4[i] : nullptr;
        const int n = n0 + a_row[i];
        w_ptr[i] = n < g.N ? g.W + (size_t)n * g.K + a_k4[i] : nullptr;
    }

    // MMA mapping: 8 warps as 2 (rows) x 4 (cols); warp tile 32 x 16 = 2 x 2 m16n8 tiles
    const int wm = warp >> 2, wn = warp & 3;
    const int gid = lane >> 2, tig = lane & 3;
    // FFMA mapping: thread tile 4 rows x 4 (strided) cols
    const int ty = tid >> 4, tx = tid & 15;

    float acc[2][2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0f;

    // operand chunks are fetched one K step ahead (registers), so the global/L2 latency of chunk
    // k+1 overlaps the tensor-core work on chunk k; small problems are pure latency otherwise
    float4 av[2], wv[2];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            av[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            wv[i] = av[i];
            const bool k_ok = k0 + a_k4[i] < g.K;
            if (a_ptr[i] && k_ok) av[i] = *reinterpret_cast<const float4 *>(a_ptr[i] + k0);
            if (w_ptr[i] && k_ok) wv[i] = __ldg(reinterpret_cast<const float4 *>(w_ptr[i] + k0));
        }
    };
    fetch(0);
    for (int k0 = 0; k0 < g.K; k0 += GEMM_BK) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            float4 a = av[i];
            if (PRO == PRO_SILU) {
                a.x = nnp_silu(a.x);
                a.y = nnp_silu(a.y);
                a.z = nnp_silu(a.z);
                a.w = nnp_silu(a.w);
            }
            *reinterpret_cast<float4 *>(&As[a_row[i]][a_k4[i]]) = a;
            *reinterpret_cast<float4 *>(&Ws[a_row[i]][a_k4[i]]) = wv[i];
        }
        if (k0 + GEMM_BK < g.K) fetch(k0 + GEMM_BK);
        __syncthreads();
        if (MMA) {
#pragma unroll
            for (int kk = 0; kk < GEMM_BK; kk += 8) {
                uint32_t ah[2][4], al[2][4], bh[2][2], bl[2][2];
#pragma unroll
                for (int mi = 0; mi < 2; ++mi) {
                    const int rb = wm * 32 + mi * 16;
                    tf32_split(As[rb + gid][kk + tig], ah[mi][0], al[mi][0]);
                    tf32_split(As[rb + gid + 8][kk + tig], ah[mi][1], al[mi][1]);
                    tf32_split(As[rb + gid][kk + tig + 4], ah[mi][2], al[mi][2]);
                    tf32_split(As[rb + gid + 8][kk + tig + 4], ah[mi][3], al[mi][3]);
                }
#pragma unroll
                for (int ni = 0; ni < 2; ++ni) {
                    const int cb = wn * 16 + ni * 8;
                    tf32_split(Ws[cb + gid][kk + tig], bh[ni][0], bl[ni][0]);
                    tf32_split(Ws[cb + gid][kk + tig + 4], bh[ni][1], bl[ni][1]);
                }
#pragma unroll
                for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 2; ++ni) {
                        // The tensor core adds into its accumulator with truncation: chaining all K
                        // steps inside it shrinks every output by ~1e-6 relative (measured: a
                        // systematic 5e-6 energy error).  Each K step therefore starts from zero and
                        // is added to the running sum by an ordinary round-to-nearest FADD.
                        float t[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                        mma_tf32(t, al[mi], bh[ni]);
                        mma_tf32(t, ah[mi], bl[ni]);
                        mma_tf32(t, ah[mi], bh[ni]);
#pragma unroll
                        for (int q = 0; q < 4; ++q) acc[mi][ni][q] += t[q];
                    }
            }
        } else {
            // acc[i>>1][i&1][j] holds row ty*4+i, col tx+16*j
#pragma unroll 8
            for (int kk = 0; kk < GEMM_BK; ++kk) {
                float a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = As[ty * 4 + i][kk];
#pragma unroll
                for (int j = 0; j < 4; ++j) b[j] = Ws[tx + 16 * j][kk];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i >> 1][i & 1][j] += a[i] * b[j];
            }
        }
        __syncthreads();
    }

    if (MMA) {
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) {
                const int r = m0 + wm * 32 + mi * 16 + gid;
                const int c = n0 + wn * 16 + ni * 8 + tig * 2;
                gemm_epilogue<EPI>(g, r, c, acc[mi][ni][0]);
                gemm_epilogue<EPI>(g, r, c + 1, acc[mi][ni][1]);
                gemm_epilogue<EPI>(g, r + 8, c, acc[mi][ni][2]);
                gemm_epilogue<EPI>(g, r + 8, c + 1, acc[mi][ni][3]);
            }
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
                gemm_epilogue<EPI>(g, m0 + ty * 4 + i, n0 + tx + 16 * j, acc[i >> 1][i & 1][j]);
    }
}

// GEMM engine of the calling thread's current library call (set at every entry point from the
// model's gemm_mode, else from the process default of nnp_set_gemm_mode):
// 5 = streaming tcgen05 for the 128 x 128 mixes, per-tile tcgen05 otherwise (default);
// 3 = per-tile tcgen05 3xTF32; 1 = mma.sync 3xTF32; 0 = FP32 FFMA
extern thread_local int t_nnp_gemm_mode;
