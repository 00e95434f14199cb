// TensorNet energy-and-forces step on sm_100a (oracle/tensornet_oracle.py
// `energy_forces_compact` is the CPU statement of exactly this arithmetic).
//
// Replaces GraphPotential.evaluate = forward + backward_forces (graphnet.py:317-412, 516-537,
// 567-580) with the TensorNet arithmetic.  Forces come from a hand-written reverse sweep, not
// autograd; geometry derivatives are collected per directed edge (g_d = dE/dd_e, g_u = dE/du_e)
// and turned into forces by one gather over each atom's row using the reverse edge, so there is
// no atomic anywhere in the step and results are bitwise reproducible.
//
// Data layout: node tensors are [N][9][C] float32 (irreducible components, channel fastest);
// a warp owns one node and each lane C/32 consecutive channels, so every row/gather access is a
// full-width coalesced vector load.  Edges arrive CSR by receiver, sorted by (receiver, sender);
// the step re-sorts every row by distance (k_edge_order) and stores each edge's reverse edge.
// Radial functions (distance projections of the embedding, radial MLP of each layer) are read
// from per-layer cubic-Hermite tables in u = exp(cutoff_lower - d), built by the host in
// float64: they depend on the distance only, so tabulating them removes the per-edge MLP
// (135k MAC/edge/layer) from both the forward and the force pass.
#include <stdlib.h>

#include <algorithm>

#include "nnp_common.cuh"
#include "tn_gemm_tc5.cuh"
#include "tn_math.cuh"

#include <atomic>
thread_local int t_nnp_gemm_mode = 5;
static std::atomic<int> g_gemm_default{5};   // nnp_set_gemm_mode: 5 = streaming tcgen05 for the 128x128 mixes
                                             // (other shapes use 3), 3 = tcgen05 one tile per CTA, 1 = mma.sync, 0 = FFMA

namespace {

constexpr float LN_EPS = 1e-5f;
constexpr float PI_F = 3.14159265358979323846f;

template <int CPL>
__device__ __forceinline__ void ldv(const float *p, float (&v)[CPL])
{
    if constexpr (CPL == 4) {
        const float4 t = __ldg(reinterpret_cast<const float4 *>(p));
        v[0] = t.x;
        v[1] = t.y;
        v[2] = t.z;
        v[3] = t.w;
    } else if constexpr (CPL == 2) {
        const float2 t = __ldg(reinterpret_cast<const float2 *>(p));
        v[0] = t.x;
        v[1] = t.y;
    } else {
        v[0] = __ldg(p);
    }
}

template <int CPL>
__device__ __forceinline__ void stv(float *p, const float (&v)[CPL])
{
    if constexpr (CPL == 4) {
        *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else if constexpr (CPL == 2) {
        *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
    } else {
        p[0] = v[0];
    }
}

constexpr int NNP_PARTS = 4;  // max channel parts a node's row is split over (C / (32 * CPL))
constexpr int NNP_GD_SLOTS = 8;

struct TnDev {
    nnp_tn_model m;
    int n, n_samples, capacity;
    int nparts;  // channel-part slots of g_u in use this step (<= NNP_PARTS)
    int gd_slots;  // g_d slots per writing kernel (<= NNP_GD_SLOTS): channel parts, times two when the
                   // reverse message kernel runs as two warps (I+A | S) per receiver
    // inputs
    const int *species, *batch, *order, *row_ptr, *pairs, *nl_counts;
    const float *deltas, *dists;
    // outputs
    float *energy, *forces, *per_atom;
    // workspace: edges (model order: CSR by receiver, each row sorted by table coordinate)
    int *col, *rev, *newpos;
    float4 *geoA;  // (table coordinate, phi, dphi/dd, 1/d)
    float4 *geoB;  // (ux, uy, uz, u = exp(cutoff_lower - d))
    // per-edge records of the interaction layers' row walkers, fixed for the whole step (every layer
    // of both sweeps reads them): sender and knot interval, and the four cubic-Hermite weights of
    // the interval's two knots, already multiplied by the cosine envelope and stored in the order
    // (even knot value, even knot slope, odd knot value, odd knot slope) - the walkers keep the
    // even-numbered and the odd-numbered knot of their current interval in two fixed register sets,
    // so moving to the next interval replaces one set and never moves data between registers.
    int2 *ejk;     // (sender j, knot interval kn)
    float4 *hwV;   // weights of f_e * phi_e
    float4 *hwD;   // weights of d(f_e * phi_e)/dd = f' * dtx/dd * phi + f * phi'
    int *ezs;      // species of the edge's sender (the embedding reads z_send[ezs[e]])
    float *g_d;    // [(L+1) * gd_slots][capacity] dE/dd_e: one slot per (writing kernel, channel part), so every
                   // kernel stores its share without a read-modify-write; summed in k_forces
    float4 *g_u;   // [NNP_PARTS][capacity] dE/du_e
    // workspace: nodes
    int *zs, *sample_ptr;
    float *X0, *n0, *ln0, *e0, *se0, *e1, *Xm, *Xa, *Xb;   // se0 = silu(e0), sr0 = silu(r0)
    float *Xh[NNP_TN_MAX_LAYERS], *nx[NNP_TN_MAX_LAYERS], *Yc[NNP_TN_MAX_LAYERS],
        *Mc[NNP_TN_MAX_LAYERS], *Dc[NNP_TN_MAX_LAYERS];
    float *Qc, *lnr, *r0, *sr0, *r1, *e_atom;
    float *G1, *G2, *G3;  // [N,9,C] gradient scratch
    float *g_r1, *g_r0, *g_lnr, *g_e1, *g_e0, *g_ln0;
    // embedding reverse by node-level projection (NULL when the model does not ask for it)
    int *present;       // [max_z] species seen this step
    int *slot_of_z;     // [max_z] slot (0..3) of a present species, in increasing species order
    int *slot_species;  // [EMB_SLOTS] species of a slot, -1 when unused
    int *embed_fast;    // [1] 1 = this step has at most EMB_SLOTS species: the projected kernels run
    float *Wproj;       // [3 groups][sender | receiver][EMB_SLOTS * 32][C] species-weighted dp weights
    float *Hb;          // [N][EMB_SLOTS * 9] bias column of the projection
};

constexpr int EMB_SLOTS = 4;   // species slots of the projected embedding reverse (EMB_SLOTS * 32 = 128 GEMM columns)
constexpr int EMB_K = 32;      // radial basis size it is written for

__device__ __forceinline__ bool overflowed(const TnDev &d)
{
    return d.nl_counts != nullptr && d.nl_counts[0] > d.capacity;
}

// ------------------------------------------------------------------------------- setup
__global__ void k_prep_nodes(TnDev d)
{
    NNP_PDL_SYNC();
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (d.present)
        for (int z = s; z < d.m.max_z; z += gridDim.x * blockDim.x) d.present[z] = 0;
    if (s >= d.n) return;
    const int i = d.order ? d.order[s] : s;
    d.zs[s] = d.species[i];
    // sample_ptr[b] = first atom of sample b (batch is non-decreasing, original order; s doubles as an
    // original index here).  Every entry is written exactly once: the codes (prev, b] start at s
    // (empty samples in between included), the codes past the last atom's end at n.
    const int b = d.batch[s];
    const int prev = s == 0 ? -1 : d.batch[s - 1];
    for (int c = prev + 1; c <= b; ++c) d.sample_ptr[c] = s;
    if (s == d.n - 1)
        for (int c = b + 1; c <= d.n_samples; ++c) d.sample_ptr[c] = d.n;
}

__device__ __forceinline__ int knot_of(float tx, int num_knots, float &t)
{
    int kn = (int)tx;
    kn = kn > num_knots - 2 ? num_knots - 2 : kn;
    t = tx - (float)kn;
    return kn;
}

// Per-edge geometry shared by every layer of the forward and reverse sweeps, written in the
// MODEL's edge order: each receiver's row is re-sorted by decreasing distance (= increasing table
// coordinate), so that consecutive edges of a row fall into the same or the next knot interval
// and the row-walking kernels keep the interval's table data in registers.  One warp per row;
// the rank of an edge inside its row is found by counting (rows are a few dozen edges).
// cosine cutoff as radial.py:11-39, u as radial.py:57.
__global__ void __launch_bounds__(256) k_edge_order(TnDev d)
{
    NNP_PDL_SYNC();
    if (overflowed(d)) return;
    const int lane = threadIdx.x & 31;
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= d.n) return;
    const int e0 = d.row_ptr[s], e1 = d.row_ptr[s + 1];
    const float rl = d.m.cutoff_lower, ru = d.m.cutoff_upper;
    if (d.present && lane == 0) d.present[d.zs[s]] = 1;   // (same value from every writer)
    for (int e = e0 + lane; e < e1; e += 32) {
        const float dist = d.dists[e];
        int rank = 0;
        for (int b = e0; b < e1; ++b) {
            const float db = __ldg(d.dists + b);
            rank += (db > dist || (db == dist && b < e)) ? 1 : 0;
        }
        const int p = e0 + rank;
        const int i = d.pairs[2 * (size_t)e], j = d.pairs[2 * (size_t)e + 1];
        const bool loop = (i == j);
        float phi, dphi;
        if (rl == 0.0f) {
            const float x = dist / ru;
            phi = dist <= ru ? 0.5f * (cospif(x) + 1.0f) : 0.0f;
            dphi = dist <= ru ? -0.5f * PI_F / ru * sinpif(x) : 0.0f;
        } else {
            const float span = ru - rl;
            const float t = 2.0f * (dist - rl) / span + 1.0f;
            const bool in = dist >= rl && dist <= ru;
            phi = in ? 0.5f * (cospif(t) + 1.0f) : 0.0f;
            dphi = in ? -PI_F / span * sinpif(t) : 0.0f;
        }
        const float u = expf(rl - dist);
        float tx = (u - d.m.u_min) / d.m.u_step;
        tx = fminf(fmaxf(tx, 0.0f), (float)(d.m.num_knots - 1));
        const float invd = loop ? 0.0f : 1.0f / dist;
        d.newpos[e] = p;
        d.col[p] = j;
        d.geoA[p] = make_float4(tx, phi, dphi, invd);
        {
            float t;
            const int kn = knot_of(tx, d.m.num_knots, t);
            const Hermite h = hermite_weights(t);
            const float su = -u / d.m.u_step * phi;            // d(table coordinate)/dd, times the envelope
            const float l0 = h.h00 * phi, l1 = h.h10 * phi, r0 = h.h01 * phi, r1 = h.h11 * phi;
            const float dl0 = fmaf(h.d00, su, h.h00 * dphi), dl1 = fmaf(h.d10, su, h.h10 * dphi);
            const float dr0 = fmaf(h.d01, su, h.h01 * dphi), dr1 = fmaf(h.d11, su, h.h11 * dphi);
            const bool even = (kn & 1) == 0;                   // the interval's left knot is the even one
            d.ejk[p] = make_int2(j, kn);
            d.ezs[p] = d.zs[j];
            d.hwV[p] = even ? make_float4(l0, l1, r0, r1) : make_float4(r0, r1, l0, l1);
            d.hwD[p] = even ? make_float4(dl0, dl1, dr0, dr1) : make_float4(dr0, dr1, dl0, dl1);
        }
        d.geoB[p] = make_float4(d.deltas[3 * (size_t)e] * invd, d.deltas[3 * (size_t)e + 1] * invd,
                                d.deltas[3 * (size_t)e + 2] * invd, u);
        for (int q = 0; q < d.nparts; ++q) d.g_u[(size_t)q * d.capacity + p] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = 0; q < d.gd_slots * (d.m.num_layers + 1); ++q) d.g_d[(size_t)q * d.capacity + p] = 0.0f;
    }
}

// rev[e] = model-order index of the reverse edge (j <- i) of e = (i <- j): bisection in the
// sender's row of the caller's list (sorted by sender), mapped through newpos.
__global__ void k_edge_rev(TnDev d)
{
    NNP_PDL_SYNC();
    if (overflowed(d)) return;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= d.row_ptr[d.n]) return;
    const int i = d.pairs[2 * (size_t)e], j = d.pairs[2 * (size_t)e + 1];
    int lo = d.row_ptr[j], hi = d.row_ptr[j + 1] - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (d.pairs[2 * (size_t)mid + 1] < i) lo = mid + 1; else hi = mid;
    }
    d.rev[d.newpos[e]] = d.newpos[lo];
}

// Radial tables come in two layouts: per knot the values and (knot-spacing-scaled) slopes of the 3
// radial functions, [knot][value|slope][3][C] (`tables`, for row walkers that keep the two knots of
// their current interval in registers), and per knot interval the monomial coefficients
// (`tables_mono`, Horner form for kernels that visit intervals in no particular order).

// Lookup of the 3 radial functions of `CPL` channels: value f[k][v] and d f / d(knot coordinate).
// The host stores, per knot interval, the cubic's monomial coefficients [c0 c1 c2 c3][3][C]
// (the Hermite interpolant of values and slopes, expanded in float64), so the device evaluates
// by Horner: f = ((c3 t + c2) t + c1) t + c0,  f' = (3 c3 t + 2 c2) t + c1.
template <int C, int CPL, bool DERIV>
__device__ __forceinline__ void table_lookup(const float *__restrict__ tab, int num_knots, float tx,
                                             int cb, float (&f)[3][CPL], float (&df)[3][CPL])
{
    int kn = (int)tx;
    kn = kn > num_knots - 2 ? num_knots - 2 : kn;
    const float t = tx - (float)kn;
    const float *row = tab + (size_t)kn * (12 * C) + cb;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float c0[CPL], c1[CPL], c2[CPL], c3[CPL];
        ldv<CPL>(row + k * C, c0);
        ldv<CPL>(row + (3 + k) * C, c1);
        ldv<CPL>(row + (6 + k) * C, c2);
        ldv<CPL>(row + (9 + k) * C, c3);
#pragma unroll
        for (int v = 0; v < CPL; ++v) {
            f[k][v] = fmaf(fmaf(fmaf(c3[v], t, c2[v]), t, c1[v]), t, c0[v]);
            if (DERIV) df[k][v] = fmaf(fmaf(3.0f * c3[v], t, 2.0f * c2[v]), t, c1[v]);
        }
    }
}

// one of the three radial functions (group k) at an already-split knot coordinate (kn, t)
template <int C, int CPL>
__device__ __forceinline__ void table_lookup_group(const float *__restrict__ tab, int kn, float t,
                                                   int cb, int k, float (&f)[CPL], float (&df)[CPL])
{
    const float *row = tab + (size_t)kn * (12 * C) + cb + k * C;
    float c0[CPL], c1[CPL], c2[CPL], c3[CPL];
    ldv<CPL>(row, c0);
    ldv<CPL>(row + 3 * C, c1);
    ldv<CPL>(row + 6 * C, c2);
    ldv<CPL>(row + 9 * C, c3);
#pragma unroll
    for (int v = 0; v < CPL; ++v) {
        f[v] = fmaf(fmaf(fmaf(c3[v], t, c2[v]), t, c1[v]), t, c0[v]);
        df[v] = fmaf(fmaf(3.0f * c3[v], t, 2.0f * c2[v]), t, c1[v]);
    }
}

__device__ __forceinline__ int group_of(int q) { return q == 0 ? 0 : (q < 4 ? 1 : 2); }

// Species slots of the projected embedding reverse.  Every block recomputes the slot table from the
// species marked present (increasing species order; at most EMB_SLOTS, else the step falls back to
// the per-channel kernel), block 0 publishes it, and block (group, side, slot) writes its 32 rows of
//   Wproj[group][side][slot * 32 + k][c] = ztab_side[species(slot)][c] * dp_wT[group][k][c]
// (side 0: sender table z_send, side 1: receiver table z_recv), the GEMM weights that contract
// dE/dX0 over channels for every (species, radial basis function).
__global__ void __launch_bounds__(256) k_embed_slots(TnDev d)
{
    NNP_PDL_SYNC();
    __shared__ int sp[EMB_SLOTS];
    const int C = d.m.channels;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        if (lane < EMB_SLOTS) sp[lane] = -1;
        __syncwarp();
        int count = 0;
        for (int base = 0; base < d.m.max_z; base += 32) {
            const int z = base + lane;
            const bool p = z < d.m.max_z && d.present[z] != 0;
            const unsigned b = __ballot_sync(NNP_FULL_MASK, p);
            const int slot = count + __popc(b & ((1u << lane) - 1u));
            if (p && slot < EMB_SLOTS) sp[slot] = z;
            if (blockIdx.x == 0 && z < d.m.max_z) d.slot_of_z[z] = (p && slot < EMB_SLOTS) ? slot : 0;
            count += __popc(b);
        }
        __syncwarp();
        if (blockIdx.x == 0) {
            if (lane < EMB_SLOTS) d.slot_species[lane] = sp[lane];
            if (lane == 0) d.embed_fast[0] = count <= EMB_SLOTS ? 1 : 0;
        }
    }
    __syncthreads();
    const int slot = blockIdx.x % EMB_SLOTS, side = (blockIdx.x / EMB_SLOTS) & 1, grp = blockIdx.x / (2 * EMB_SLOTS);
    const int z = sp[slot];
    const float *ztab = (side ? d.m.z_recv : d.m.z_send) + (size_t)(z < 0 ? 0 : z) * C;
    const float *w = d.m.dp_wT + (size_t)grp * EMB_K * C;
    float *out = d.Wproj + ((size_t)(grp * 2 + side) * EMB_SLOTS + slot) * EMB_K * C;
    for (int idx = threadIdx.x; idx < EMB_K * C; idx += blockDim.x) {
        const int c = idx % C;
        out[idx] = z < 0 ? 0.0f : ztab[c] * w[idx];
    }
}

// ----------------------------------------------------------------------------- embedding
// X0_i = sum_e w_e[:,grp] * basis_e  with w_e = dp(rho_e) * phi_e * Z_e ; then n0 = |X0|^2 and
// ln0 = LayerNorm_C(n0).
template <int C, int CPL>
__global__ void __launch_bounds__(256) k_embed_edge(TnDev d)
{
    NNP_PDL_SYNC();
    constexpr int NPARTS = C / (32 * CPL);
    if (overflowed(d)) return;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int s = gw / NPARTS, part = gw - s * NPARTS;
    if (s >= d.n) return;
    const int cb = part * 32 * CPL + lane * CPL;
    float zr[CPL];
    ldv<CPL>(d.m.z_recv + (size_t)d.zs[s] * C + cb, zr);
    float acc[9][CPL];
#pragma unroll
    for (int q = 0; q < 9; ++q)
#pragma unroll
        for (int v = 0; v < CPL; ++v) acc[q][v] = 0.0f;

    const int e0 = d.row_ptr[s], e1 = d.row_ptr[s + 1];
    for (int e = e0; e < e1; ++e) {
        const int j = d.col[e];
        const float4 ga = d.geoA[e];
        const float4 gb = d.geoB[e];
        float zsnd[CPL];
        ldv<CPL>(d.m.z_send + (size_t)d.zs[j] * C + cb, zsnd);
        float f[3][CPL], df[3][CPL];
        table_lookup<C, CPL, false>(d.m.tables_mono, d.m.num_knots, ga.x, cb, f, df);
        float b[9];
        edge_basis9(gb.x, gb.y, gb.z, b);
#pragma unroll
        for (int v = 0; v < CPL; ++v) {
            const float cc = ga.y * (zr[v] + zsnd[v]);
            const float w0 = f[0][v] * cc, w1 = f[1][v] * cc, w2 = f[2][v] * cc;
            acc[0][v] += w0;
#pragma unroll
            for (int q = 1; q < 4; ++q) acc[q][v] += w1 * b[q];
#pragma unroll
            for (int q = 4; q < 9; ++q) acc[q][v] += w2 * b[q];
        }
    }
    float nrm[CPL];
#pragma unroll
    for (int v = 0; v < CPL; ++v) {
        float c9[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) c9[q] = acc[q][v];
        nrm[v] = c9_frob(c9, c9);
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) stv<CPL>(d.X0 + ((size_t)s * 9 + q) * C + cb, acc[q]);
    stv<CPL>(d.n0 + (size_t)s * C + cb, nrm);
}

// ln0 = LayerNorm_C(n0): one warp per node over all channels
template <int C>
__global__ void __launch_bounds__(256) k_embed_ln(TnDev d)
{
    NNP_PDL_SYNC();
    constexpr int CPL = C / 32;
    const int lane = threadIdx.x & 31;
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= d.n) return;
    const int cb = lane * CPL;
    float nrm[CPL];
    ldv<CPL>(d.n0 + (size_t)s * C + cb, nrm);
    float sum = 0.0f;
#pragma unroll
    for (int v = 0; v < CPL; ++v) sum += nrm[v];
    const float mean = nnp_warp_sum(sum) * (1.0f / C);
    float var = 0.0f;
#pragma unroll
    for (int v = 0; v < CPL; ++v) var += (nrm[v] - mean) * (nrm[v] - mean);
    var = nnp_warp_sum(var) * (1.0f / C);
    const float rstd = rsqrtf(var + LN_EPS);
    float g[CPL], bb[CPL], out[CPL];
    ldv<CPL>(d.m.init_norm_g + cb, g);
    ldv<CPL>(d.m.init_norm_b + cb, bb);
#pragma unroll
    for (int v = 0; v < CPL; ++v) out[v] = (nrm[v] - mean) * rstd * g[v] + bb[v];
    stv<CPL>(d.ln0 + (size_t)s * C + cb, out);
}

// ------------------------------------------------------------------------- elementwise
// one thread per (node, channel); the 9 components are C floats apart
__device__ __forceinline__ void ld9(const float *base, int C, float *c9)
{
#pragma unroll
    for (int q = 0; q < 9; ++q) c9[q] = base[(size_t)q * C];
}
__device__ __forceinline__ void st9(float *base, int C, const float *c9)
{
#pragma unroll
    for (int q = 0; q < 9; ++q) base[(size_t)q * C] = c9[q];
}

// Xh = X / (|X|^2 + 1); with e1 != NULL the input is the embedding's mixed tensor Xm and
// X = Xm * silu(e1)[grp] is formed on the fly (the gated X itself is never stored)
__global__ void k_normalize(const float *__restrict__ X, const float *__restrict__ e1,
                            float *__restrict__ Xh, float *__restrict__ nx, int n, int C)
{
    NNP_PDL_SYNC();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * C) return;
    const int node = idx / C, c = idx - node * C;
    const size_t off = (size_t)node * 9 * C + c;
    float x[9], xh[9];
    ld9(X + off, C, x);
    if (e1) {
        const float *e = e1 + (size_t)node * 3 * C + 3 * c;
        const float gate[3] = {nnp_silu(e[0]), nnp_silu(e[1]), nnp_silu(e[2])};
#pragma unroll
        for (int q = 0; q < 9; ++q) x[q] *= gate[group_of(q)];
    }
    nx[idx] = normalize_fwd(x, xh);
    st9(Xh + off, C, xh);
}

// X_new = Xh + D + D*D, written either as X_new (last layer, read by the head) or directly as the
// next layer's normalised input Xh' = X_new / (|X_new|^2 + 1) together with that norm.
__global__ void k_residual(const float *__restrict__ Xh, const float *__restrict__ Dc,
                           float *__restrict__ Xn, float *__restrict__ Xh_next,
                           float *__restrict__ nx_next, int n, int C)
{
    NNP_PDL_SYNC();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * C) return;
    const int node = idx / C, c = idx - node * C;
    const size_t off = (size_t)node * 9 * C + c;
    float xh[9], dc[9], xn[9];
    ld9(Xh + off, C, xh);
    ld9(Dc + off, C, dc);
    residual_fwd(xh, dc, xn);
    if (Xh_next) {
        float nh[9];
        nx_next[idx] = normalize_fwd(xn, nh);
        st9(Xh_next + off, C, nh);
    } else {
        st9(Xn + off, C, xn);
    }
}

__global__ void k_node_product_bwd(const float *__restrict__ Mc, const float *__restrict__ Yc,
                                   const float *__restrict__ GQ, float *__restrict__ GM,
                                   float *__restrict__ GY, int n, int C)
{
    NNP_PDL_SYNC();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * C) return;
    const int node = idx / C, c = idx - node * C;
    const size_t off = (size_t)node * 9 * C + c;
    float m[9], y[9], gq[9], gm[9], gy[9];
    ld9(Mc + off, C, m);
    ld9(Yc + off, C, y);
    ld9(GQ + off, C, gq);
    node_product_bwd(m, y, gq, gm, gy);
    st9(GM + off, C, gm);
    st9(GY + off, C, gy);
}

// dL/dXh arrives in two parts (the residual path GXa and the mixed-back edge path GXb).  What
// consumes dL/dX next is fused in, so the gradient makes one trip through HBM instead of two:
//   * Dc_prev != NULL (layer l >= 1): also G_D = GX + GX*D^T + D^T*GX of layer l - 1 (k_residual_bwd);
//   * Xm != NULL (layer 0): X = Xm * silu(e1)[grp] (k_embed_gate_bwd): G_Xm = GX * gate and
//     g_e1 = <GX, Xm>_grp * silu'(e1) are written INSTEAD of GX, which nothing else reads.
__global__ void k_normalize_bwd(const float *GXa, const float *__restrict__ GXb,
                                const float *__restrict__ Xh, const float *__restrict__ nx,
                                float *GX /* may alias GXa: every thread reads its own nine values first */,
                                const float *__restrict__ Dc_prev,
                                float *__restrict__ GD, const float *__restrict__ Xm,
                                const float *__restrict__ e1, float *__restrict__ GXm,
                                float *__restrict__ g_e1, int n, int C)
{
    NNP_PDL_SYNC();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * C) return;
    const int node = idx / C, c = idx - node * C;
    const size_t off = (size_t)node * 9 * C + c;
    float g[9], g2[9], xh[9], gx[9];
    ld9(GXa + off, C, g);
    ld9(GXb + off, C, g2);
#pragma unroll
    for (int q = 0; q < 9; ++q) g[q] += g2[q];
    ld9(Xh + off, C, xh);
    normalize_bwd(g, xh, nx[idx], gx);
    if (Xm) {
        float xm[9], gxm[9];
        ld9(Xm + off, C, xm);
        const float *e = e1 + (size_t)node * 3 * C + 3 * c;
        const float gate[3] = {nnp_silu(e[0]), nnp_silu(e[1]), nnp_silu(e[2])};
#pragma unroll
        for (int q = 0; q < 9; ++q) gxm[q] = gx[q] * gate[group_of(q)];
        st9(GXm + off, C, gxm);
        float *ge = g_e1 + (size_t)node * 3 * C + 3 * c;
        ge[0] = c9_dot_I(gx, xm) * nnp_silu_grad(e[0]);
        ge[1] = c9_dot_A(gx, xm) * nnp_silu_grad(e[1]);
        ge[2] = c9_dot_S(gx, xm) * nnp_silu_grad(e[2]);
        return;
    }
    st9(GX + off, C, gx);
    if (Dc_prev) {
        float dc[9], gd[9];
        ld9(Dc_prev + off, C, dc);
        residual_bwd(gx, dc, gd);
        st9(GD + off, C, gd);
    }
}

// X = Xm * gate[grp], gate = silu(e1):  G_Xm = GX*gate ; g_e1 = <GX, Xm>_grp * silu'(e1)
__global__ void k_embed_gate_bwd(const float *__restrict__ GX, const float *__restrict__ Xm,
                                 const float *__restrict__ e1, float *__restrict__ GXm,
                                 float *__restrict__ g_e1, int n, int C)
{
    NNP_PDL_SYNC();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * C) return;
    const int node = idx / C, c = idx - node * C;
    const size_t off = (size_t)node * 9 * C + c;
    float g[9], xm[9], gxm[9];
    ld9(GX + off, C, g);
    ld9(Xm + off, C, xm);
    const float *e = e1 + (size_t)node * 3 * C + 3 * c;
    const float gate[3] = {nnp_silu(e[0]), nnp_silu(e[1]), nnp_silu(e[2])};
#pragma unroll
    for (int q = 0; q < 9; ++q) gxm[q] = g[q] * gate[group_of(q)];
    st9(GXm + off, C, gxm);
    float *ge = g_e1 + (size_t)node * 3 * C + 3 * c;
    ge[0] = c9_dot_I(g, xm) * nnp_silu_grad(e[0]);
    ge[1] = c9_dot_A(g, xm) * nnp_silu_grad(e[1]);
    ge[2] = c9_dot_S(g, xm) * nnp_silu_grad(e[2]);
}

// ----------------------------------------------------------------------- interaction edges
// The two knots of a row walker's current table interval, for the radial functions [K0, K0 + NG),
// held in two fixed register sets: the even-numbered knot and the odd-numbered knot.  Rows are
// sorted by table coordinate, so moving on means "same interval" (nothing), "next interval" (one
// knot replaces the one that fell behind - no register moves, the per-edge weights of k_edge_order
// already come in (even, odd) order) or a jump (both knots) - a warp-uniform decision.
template <int C, int CPL, int K0, int NG>
struct KnotEO {
    float ev[NG][CPL], em[NG][CPL], ov[NG][CPL], om[NG][CPL];
    int kn;
    __device__ __forceinline__ void init() { kn = -4; }
    __device__ __forceinline__ static void load_knot(const float *__restrict__ tab, int knot, int cb,
                                                     float (&v)[NG][CPL], float (&m)[NG][CPL])
    {
        const float *row = tab + (size_t)knot * (6 * C) + cb;
#pragma unroll
        for (int k = 0; k < NG; ++k) {
            ldv<CPL>(row + (K0 + k) * C, v[k]);
            ldv<CPL>(row + (3 + K0 + k) * C, m[k]);
        }
    }
    __device__ __forceinline__ void seek(const float *__restrict__ tab, int k, int cb)
    {
        if (k == kn) return;
        const bool jump = k != kn + 1;
        if (k & 1) {                       // left knot k is odd, right knot k + 1 even
            if (jump) load_knot(tab, k, cb, ov, om);
            load_knot(tab, k + 1, cb, ev, em);
        } else {
            if (jump) load_knot(tab, k, cb, ev, em);
            load_knot(tab, k + 1, cb, ov, om);
        }
        kn = k;
    }
    // w = the edge's four weights in (even value, even slope, odd value, odd slope) order
    __device__ __forceinline__ void eval(const float4 &w, int k, float (&f)[CPL]) const
    {
#pragma unroll
        for (int v = 0; v < CPL; ++v)
            f[v] = fmaf(w.x, ev[k][v], fmaf(w.y, em[k][v], fmaf(w.z, ov[k][v], w.w * om[k][v])));
    }
};

// The embedding's edge sum as two knot-cached warps per (receiver, channel part), like the message
// kernel: X0_i[q] = sum_e (dp_g(q)(d_e) phi_e) (z_recv[z_i] + z_send[z_j]) b_q(u_e).  The radial part
// comes from the interval's two knots in registers and the per-edge weights of k_edge_order (table 0,
// envelope folded in), the species factor from the sender-species record, so an edge costs one
// 16-byte table-row read instead of twelve coefficient loads.
template <int C, int CPL, int K0, int NG, int Q0, int NQ>
__device__ __forceinline__ void embed_row_part(const TnDev &d, int s, int cb, float (&acc)[NQ][CPL])
{
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int v = 0; v < CPL; ++v) acc[q][v] = 0.0f;
    float zr[CPL];
    ldv<CPL>(d.m.z_recv + (size_t)d.zs[s] * C + cb, zr);
    const float *tab = d.m.tables;                      // table 0: the three distance projections
    const int e0 = d.row_ptr[s], e1 = d.row_ptr[s + 1];
    KnotEO<C, CPL, K0, NG> kc;
    kc.init();
    const int2 *__restrict__ ejk = d.ejk;
    const float4 *__restrict__ hwV = d.hwV;
    const float4 *__restrict__ geoB = d.geoB;
    const int *__restrict__ ezs = d.ezs;
    const float *zsend = d.m.z_send + cb;
    int kn = e0 < e1 ? __ldg(ejk + e0).y : 0;
    int zj = e0 < e1 ? __ldg(ezs + e0) : 0;
    for (int e = e0; e < e1; ++e) {
        float zs[CPL];
        ldv<CPL>(zsend + (size_t)zj * C, zs);
        const float4 wc = __ldg(hwV + e);
        const float4 gb = __ldg(geoB + e);
        kc.seek(tab, kn, cb);
        if (e + 1 < e1) {
            kn = __ldg(ejk + e + 1).y;
            zj = __ldg(ezs + e + 1);
        }
        float b[9];
        edge_basis9(gb.x, gb.y, gb.z, b);
#pragma unroll
        for (int k = 0; k < NG; ++k) {
            float f[CPL];
            kc.eval(wc, k, f);
#pragma unroll
            for (int v = 0; v < CPL; ++v) f[v] *= zr[v] + zs[v];
            const int g = K0 + k;
            const int qa = (g == 0 ? 0 : (g == 1 ? 1 : 4)), qb = (g == 0 ? 1 : (g == 1 ? 4 : 9));
#pragma unroll
            for (int q = qa; q < qb; ++q)
#pragma unroll
                for (int v = 0; v < CPL; ++v) acc[q - Q0][v] = fmaf(f[v], b[q], acc[q - Q0][v]);
        }
    }
    float *out = d.X0 + ((size_t)s * 9 + Q0) * C + cb;
#pragma unroll
    for (int q = 0; q < NQ; ++q) stv<CPL>(out + q * C, acc[q]);
}

// launched with blocks of 64 * k threads: the two halves of a (receiver, part) are neighbouring warps
template <int C, int CPL>
__global__ void __launch_bounds__(128, 5) k_embed_edge_split(TnDev d)
{
    NNP_PDL_SYNC();
    constexpr int NPARTS = C / (32 * CPL);
    __shared__ float s_norm[4][32 * CPL];               // S-half partial of |X0|^2, per warp of the block
    if (overflowed(d)) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * (blockDim.x >> 5) + wib;
    const int s = gw / (2 * NPARTS), rem = gw - s * (2 * NPARTS);
    const int part = rem >> 1, half = rem & 1;
    const bool live = s < d.n;
    const int cb = part * 32 * CPL + lane * CPL;
    float nrm[CPL];
#pragma unroll
    for (int v = 0; v < CPL; ++v) nrm[v] = 0.0f;
    if (live) {
        if (half == 0) {
            float acc[4][CPL];
            embed_row_part<C, CPL, 0, 2, 0, 4>(d, s, cb, acc);
#pragma unroll
            for (int v = 0; v < CPL; ++v)       // <X,X>_I + <X,X>_A = 3 s^2 + 2 |a|^2
                nrm[v] = 3.0f * acc[0][v] * acc[0][v] +
                         2.0f * (acc[1][v] * acc[1][v] + acc[2][v] * acc[2][v] + acc[3][v] * acc[3][v]);
        } else {
            float acc[5][CPL];
            embed_row_part<C, CPL, 2, 1, 4, 5>(d, s, cb, acc);
#pragma unroll
            for (int v = 0; v < CPL; ++v) {     // <X,X>_S with Szz = -Sxx - Syy
                const float szz = acc[0][v] + acc[1][v];
                nrm[v] = acc[0][v] * acc[0][v] + acc[1][v] * acc[1][v] + szz * szz +
                         2.0f * (acc[2][v] * acc[2][v] + acc[3][v] * acc[3][v] + acc[4][v] * acc[4][v]);
                s_norm[wib][lane * CPL + v] = nrm[v];
            }
        }
    }
    __syncthreads();
    if (live && half == 0) {
#pragma unroll
        for (int v = 0; v < CPL; ++v) nrm[v] += s_norm[wib + 1][lane * CPL + v];
        stv<CPL>(d.n0 + (size_t)s * C + cb, nrm);
    }
}

// one knot-cached warp per (receiver, part) over all nine components (three radial groups in registers)
template <int C, int CPL>
__global__ void __launch_bounds__(128, 4) k_embed_edge_knots(TnDev d)
{
    NNP_PDL_SYNC();
    constexpr int NPARTS = C / (32 * CPL);
    if (overflowed(d)) return;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int s = gw / NPARTS, part = gw - s * NPARTS;
    if (s >= d.n) return;
    const int cb = part * 32 * CPL + lane * CPL;
    float acc[9][CPL];
    embed_row_part<C, CPL, 0, 3, 0, 9>(d, s, cb, acc);
    float nrm[CPL];
#pragma unroll
    for (int v = 0; v < CPL; ++v) {
        float c9[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) c9[q] = acc[q][v];
        nrm[v] = c9_frob(c9, c9);
    }
    stv<CPL>(d.n0 + (size_t)s * C + cb, nrm);
}

// One warp's share of a receiver row: components [Q0, Q0 + NQ) = radial groups [K0, K0 + NG).
template <int C, int CPL, int K0, int NG, int Q0, int NQ>
__device__ __forceinline__ void message_row_part(const TnDev &d, const float *__restrict__ tab,
                                                 const float *__restrict__ Y, float *__restrict__ Mout,
                                                 int s, int cb)
{
    float acc[NQ][CPL];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int v = 0; v < CPL; ++v) acc[q][v] = 0.0f;
    const int e0 = d.row_ptr[s], e1 = d.row_ptr[s + 1];
    KnotEO<C, CPL, K0, NG> kc;
    kc.init();
    const int2 *__restrict__ ejk = d.ejk;
    const float4 *__restrict__ hwV = d.hwV;
    const float *ybase = Y + Q0 * C + cb;
    int2 jk = e0 < e1 ? __ldg(ejk + e0) : make_int2(0, 0);
    for (int e = e0; e < e1; ++e) {
        const float *yj = ybase + (size_t)jk.x * (9 * C);
        float y[NQ][CPL];
#pragma unroll
        for (int q = 0; q < NQ; ++q) ldv<CPL>(yj + q * C, y[q]);
        const float4 wc = __ldg(hwV + e);       // lands together with the gathered row
        kc.seek(tab, jk.y, cb);
        if (e + 1 < e1) jk = __ldg(ejk + e + 1);
#pragma unroll
        for (int k = 0; k < NG; ++k) {
            float f[CPL];
            kc.eval(wc, k, f);
            // local component range of group K0 + k
            const int g = K0 + k;
            const int qa = (g == 0 ? 0 : (g == 1 ? 1 : 4)) - Q0, qb = (g == 0 ? 1 : (g == 1 ? 4 : 9)) - Q0;
#pragma unroll
            for (int q = qa; q < qb; ++q)
#pragma unroll
                for (int v = 0; v < CPL; ++v) acc[q][v] = fmaf(f[v], y[q][v], acc[q][v]);
        }
    }
    float *out = Mout + ((size_t)s * 9 + Q0) * C + cb;
#pragma unroll
    for (int q = 0; q < NQ; ++q) stv<CPL>(out + q * C, acc[q]);
}

// M_i = sum_e f_e[:,grp] * Yc_j with two warps per (receiver, channel part): one owns the I and A
// components (4 of 9), the other the S components (5 of 9), so each keeps only its own groups'
// knot data and accumulators in registers.  The node update Q = (M*Y + Y*M)/(|.|^2 + 1) follows
// after a block barrier, the two warps taking half of the lane's channels each.
template <int C, int CPL>
__global__ void __launch_bounds__(128, 5) k_edge_message_split(TnDev d, int layer)
{
    NNP_PDL_SYNC();
    constexpr int NPARTS = C / (32 * CPL);
    if (overflowed(d)) return;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int s = gw / (2 * NPARTS), rem = gw - s * (2 * NPARTS);
    const int part = rem >> 1, half = rem & 1;
    const bool live = s < d.n;
    const int cb = part * 32 * CPL + lane * CPL;
    const float *tab = d.m.tables + (size_t)(layer + 1) * d.m.num_knots * 6 * C;
    const float *Y = d.Yc[layer];
    float *M = d.Mc[layer];
    if (live) {
        if (half == 0) message_row_part<C, CPL, 0, 2, 0, 4>(d, tab, Y, M, s, cb);
        else message_row_part<C, CPL, 2, 1, 4, 5>(d, tab, Y, M, s, cb);
    }
    __syncthreads();   // the partner warp's components of M are visible now
    if (!live) return;
    constexpr int HC = CPL >= 2 ? CPL / 2 : 1;      // channels per lane in the node update
    if (CPL == 1 && half == 1) return;
    const int cq = cb + (CPL >= 2 ? half * HC : 0);
    const float *mi = M + (size_t)s * 9 * C + cq;
    const float *yi = Y + (size_t)s * 9 * C + cq;
    float mv[9][HC], yv[9][HC], qv[9][HC];
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        if constexpr (HC == 2) {
            const float2 a = *reinterpret_cast<const float2 *>(mi + q * C);   // written this launch: no __ldg
            mv[q][0] = a.x;
            mv[q][1] = a.y;
        } else {
            mv[q][0] = mi[q * C];
        }
        ldv<HC>(yi + q * C, yv[q]);
    }
#pragma unroll
    for (int v = 0; v < HC; ++v) {
        float m9[9], y9[9], q9[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            m9[q] = mv[q][v];
            y9[q] = yv[q][v];
        }
        node_product_fwd(m9, y9, q9);
#pragma unroll
        for (int q = 0; q < 9; ++q) qv[q][v] = q9[q];
    }
    float *qo = d.Qc + (size_t)s * 9 * C + cq;
#pragma unroll
    for (int q = 0; q < 9; ++q) stv<HC>(qo + q * C, qv[q]);
}

// The same reverse edge op as k_edge_message_bwd below (see there for the formulas), run like the
// forward kernel: two warps per (receiver, channel part) - one owns the I and A components, the other
// the S components - each walking the distance-sorted row with the interval's two knots in registers
// and the per-edge Hermite weights of k_edge_order (hwV for f*phi, hwD for d(f*phi)/dd), so no table
// coefficient is loaded per edge.  The per-edge sum over channels is collected eight edges at a time:
// every lane keeps its partial of eight edges and one transposing butterfly (7 + 2 shuffles) leaves
// the eight totals in lanes 0, 4, ..., 28, which store them side by side.
template <int C, int CPL, int K0, int NG, int Q0, int NQ>
__device__ __forceinline__ void message_bwd_row_part(const TnDev &d, const float *__restrict__ tab,
                                                     const float *__restrict__ GM, float *__restrict__ GY,
                                                     const float *__restrict__ Yown, float *__restrict__ gd_slot,
                                                     int s, int cb)
{
    const int lane = threadIdx.x & 31;
    // wy[q] = weight of gathered component q in <G_M[b], Yc[a]> of its group (metric folded in):
    // I: 3 y0 ; A: 2 y_q ; S: 2 y4 + y5, 2 y5 + y4, 2 y_q
    float wy[NQ][CPL], acc[NQ][CPL];
    {
        const float *p = Yown + ((size_t)s * 9 + Q0) * C + cb;
        const float *py = GY + ((size_t)s * 9 + Q0) * C + cb;
        float y[NQ][CPL];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            ldv<CPL>(p + q * C, y[q]);
            ldv<CPL>(py + q * C, acc[q]);
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int v = 0; v < CPL; ++v) {
                const int gq = Q0 + q;
                wy[q][v] = gq == 0 ? 3.0f * y[q][v]
                         : gq == 4 ? 2.0f * y[q][v] + y[q + (gq == 4 ? 1 : 0)][v]
                         : gq == 5 ? 2.0f * y[q][v] + y[q - (gq == 5 ? 1 : 0)][v]
                                   : 2.0f * y[q][v];
            }
    }
    const int e0 = d.row_ptr[s], e1 = d.row_ptr[s + 1];
    KnotEO<C, CPL, K0, NG> kc;
    kc.init();
    const int2 *__restrict__ ejk = d.ejk;
    const float4 *__restrict__ hwV = d.hwV;
    const float4 *__restrict__ hwD = d.hwD;
    const float *gbase = GM + Q0 * C + cb;
    // MEASURED and dropped (profiles/r2_summary.md): keeping the gather of edge e + 1 in flight while
    // edge e is evaluated (second row buffer, 147 registers) - 1.68 ms per step against 1.31 ms; the same
    // with the gather requested before the knot loads 2.27 ms (loads complete in issue order).
    int2 jk = e0 < e1 ? __ldg(ejk + e0) : make_int2(0, 0);
    for (int eb = e0; eb < e1; eb += 8) {
        float pb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            pb[i] = 0.0f;
            if (eb + i < e1) {                       // warp-uniform
                float g[NQ][CPL];
                const float4 wvc = __ldg(hwV + eb + i), wdc = __ldg(hwD + eb + i);   // land with the gathered row
                const float *gj = gbase + (size_t)jk.x * (9 * C);
#pragma unroll
                for (int q = 0; q < NQ; ++q) ldv<CPL>(gj + q * C, g[q]);
                kc.seek(tab, jk.y, cb);
                if (eb + i + 1 < e1) jk = __ldg(ejk + eb + i + 1);
                float p = 0.0f;
#pragma unroll
                for (int k = 0; k < NG; ++k) {
                    float f[CPL], F[CPL], dk[CPL];
                    kc.eval(wvc, k, f);
                    kc.eval(wdc, k, F);
                    const int gi = K0 + k;
                    const int qa = (gi == 0 ? 0 : (gi == 1 ? 1 : 4)) - Q0, qb = (gi == 0 ? 1 : (gi == 1 ? 4 : 9)) - Q0;
#pragma unroll
                    for (int v = 0; v < CPL; ++v) dk[v] = 0.0f;
#pragma unroll
                    for (int q = qa; q < qb; ++q)
#pragma unroll
                        for (int v = 0; v < CPL; ++v) {
                            acc[q][v] = fmaf(f[v], g[q][v], acc[q][v]);
                            dk[v] = fmaf(g[q][v], wy[q][v], dk[v]);
                        }
#pragma unroll
                    for (int v = 0; v < CPL; ++v) p = fmaf(dk[v], F[v], p);
                }
                pb[i] = p;
            }
        }
        // eight warp sums at once: after the three transposing steps lane l holds (a quarter of) the
        // total of edge ((l >> 4) & 1) * 4 + ((l >> 3) & 1) * 2 + ((l >> 2) & 1)
#pragma unroll
        for (int o = 16, h = 4; h >= 1; o >>= 1, h >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < h; ++i) {
                const float send = up ? pb[i] : pb[i + h];
                const float keep = up ? pb[i + h] : pb[i];
                pb[i] = keep + __shfl_xor_sync(NNP_FULL_MASK, send, o);
            }
        }
        float tot = pb[0];
        tot += __shfl_xor_sync(NNP_FULL_MASK, tot, 2);
        tot += __shfl_xor_sync(NNP_FULL_MASK, tot, 1);
        const int idx = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
        if ((lane & 3) == 0 && eb + idx < e1 && __ldg(ejk + eb + idx).x != s) gd_slot[eb + idx] = tot;
    }
    float *out = GY + ((size_t)s * 9 + Q0) * C + cb;
#pragma unroll
    for (int q = 0; q < NQ; ++q) stv<CPL>(out + q * C, acc[q]);
}

template <int C, int CPL>
__global__ void __launch_bounds__(128, 4) k_edge_message_bwd_split(TnDev d, int layer, const float *GM,
                                                                float *GY, float *gd_layer)
{
    NNP_PDL_SYNC();
    constexpr int NPARTS = C / (32 * CPL);
    if (overflowed(d)) return;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int s = gw / (2 * NPARTS), rem = gw - s * (2 * NPARTS);
    const int part = rem >> 1, half = rem & 1;
    if (s >= d.n) return;
    const int cb = part * 32 * CPL + lane * CPL;
    const float *tab = d.m.tables + (size_t)(layer + 1) * d.m.num_knots * 6 * C;
    float *gd_slot = gd_layer + (size_t)(2 * part + half) * d.capacity;   // this warp's own slots
    if (half == 0) message_bwd_row_part<C, CPL, 0, 2, 0, 4>(d, tab, GM, GY, d.Yc[layer], gd_slot, s, cb);
    else message_bwd_row_part<C, CPL, 2, 1, 4, 5>(d, tab, GM, GY, d.Yc[layer], gd_slot, s, cb);
}

// ---- sender rows through a shared-memory ring fed by bulk asynchronous copies (TMA engine)
// A block is one receiver (both component halves, all channel parts), so every warp of the block
// needs the same sender row: one elected lane requests the whole 9 x C row of the edge RING_DEPTH
// positions ahead with a single cp.async.bulk (global -> shared, completion counted on an mbarrier),
// and the warps read their components from shared memory when the row has landed.  The L2 round
// trip of the gather is then hidden behind RING_DEPTH edges of arithmetic instead of being paid per
// edge by every warp (the register-gather version sits at 44 % issue utilisation waiting on
// long-scoreboard stalls); the bytes that cross the L2 fabric are unchanged.
// MEASURED (config C, profiles/r2_summary.md): 1.06 ms per launch against 0.65 ms for the register
// gather - the bulk-copy path delivered 7.4 TB/s (19 B/clk/SM) where the LDG path reaches 16.7 TB/s,
// and the mbarrier polls add 40 % instructions.  Kept selectable (NNP_BWD_SPLIT=2), not the default.
constexpr int RING_DEPTH = 4;

__device__ __forceinline__ uint32_t ring_smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ring_bar_init(uint64_t *bar, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ring_smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void ring_bar_wait(uint64_t *bar, uint32_t parity)
{
    const uint32_t addr = ring_smem_u32(bar);
    uint32_t done = 0;
    for (long spin = 0; !done; ++spin) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (spin > (1L << 28)) __trap();   // never hang the device on a protocol error
    }
}
__device__ __forceinline__ void ring_bar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ring_smem_u32(bar)) : "memory");
}
// request `bytes` (multiple of 16, both addresses 16-byte aligned) and announce them on `bar`
__device__ __forceinline__ void ring_bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    const uint32_t b = ring_smem_u32(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(ring_smem_u32(dst)), "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}

template <int C>
struct RowRing {
    float *rows;            // [RING_DEPTH][9 * C]
    uint64_t *full, *empty; // [RING_DEPTH] each
};

template <int C, int CPL, int K0, int NG, int Q0, int NQ>
__device__ __forceinline__ void message_bwd_row_ring(const TnDev &d, const float *__restrict__ tab,
                                                     const float *__restrict__ GM, float *__restrict__ GY,
                                                     const float *__restrict__ Yown, float *__restrict__ gd_slot,
                                                     int s, int cb, const RowRing<C> &ring, bool producer)
{
    const int lane = threadIdx.x & 31;
    float wy[NQ][CPL], acc[NQ][CPL];
    {
        const float *p = Yown + ((size_t)s * 9 + Q0) * C + cb;
        const float *py = GY + ((size_t)s * 9 + Q0) * C + cb;
        float y[NQ][CPL];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            ldv<CPL>(p + q * C, y[q]);
            ldv<CPL>(py + q * C, acc[q]);
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int v = 0; v < CPL; ++v) {
                const int gq = Q0 + q;
                wy[q][v] = gq == 0 ? 3.0f * y[q][v]
                         : gq == 4 ? 2.0f * y[q][v] + y[q + (gq == 4 ? 1 : 0)][v]
                         : gq == 5 ? 2.0f * y[q][v] + y[q - (gq == 5 ? 1 : 0)][v]
                                   : 2.0f * y[q][v];
            }
    }
    const int e0 = d.row_ptr[s], e1 = d.row_ptr[s + 1];
    KnotEO<C, CPL, K0, NG> kc;
    kc.init();
    const int2 *__restrict__ ejk = d.ejk;
    const float4 *__restrict__ hwV = d.hwV;
    const float4 *__restrict__ hwD = d.hwD;
    constexpr uint32_t ROW_BYTES = 9 * C * sizeof(float);
    // prologue: the first RING_DEPTH rows are requested at once (their slots are free)
    if (producer && lane == 0) {
        for (int i = 0; i < RING_DEPTH && e0 + i < e1; ++i)
            ring_bulk_load(ring.rows + i * (9 * C), GM + (size_t)__ldg(ejk + e0 + i).x * (9 * C), ROW_BYTES,
                           ring.full + i);
    }
    int kn_next = e0 < e1 ? __ldg(ejk + e0).y : 0;
    int j_ahead = (producer && e0 + RING_DEPTH < e1) ? __ldg(ejk + e0 + RING_DEPTH).x : 0;   // sender of edge e + RING_DEPTH
    for (int eb = e0; eb < e1; eb += 8) {
        float pb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            pb[i] = 0.0f;
            if (eb + i < e1) {                       // warp-uniform
                const int idx = eb + i - e0;
                const int slot = idx % RING_DEPTH;
                const uint32_t use = (uint32_t)(idx / RING_DEPTH);
                const float4 wvc = __ldg(hwV + eb + i), wdc = __ldg(hwD + eb + i);
                const int kn = kn_next;
                kc.seek(tab, kn, cb);
                if (eb + i + 1 < e1) kn_next = __ldg(ejk + eb + i + 1).y;
                ring_bar_wait(ring.full + slot, use & 1u);
                const float *gj = ring.rows + slot * (9 * C) + Q0 * C + cb;
                float g[NQ][CPL];
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    if constexpr (CPL == 4) {
                        const float4 t = *reinterpret_cast<const float4 *>(gj + q * C);
                        g[q][0] = t.x; g[q][1] = t.y; g[q][2] = t.z; g[q][3] = t.w;
                    } else if constexpr (CPL == 2) {
                        const float2 t = *reinterpret_cast<const float2 *>(gj + q * C);
                        g[q][0] = t.x; g[q][1] = t.y;
                    } else {
                        g[q][0] = gj[q * C];
                    }
                }
                float p = 0.0f;
#pragma unroll
                for (int k = 0; k < NG; ++k) {
                    float f[CPL], F[CPL], dk[CPL];
                    kc.eval(wvc, k, f);
                    kc.eval(wdc, k, F);
                    const int gi = K0 + k;
                    const int qa = (gi == 0 ? 0 : (gi == 1 ? 1 : 4)) - Q0, qb = (gi == 0 ? 1 : (gi == 1 ? 4 : 9)) - Q0;
#pragma unroll
                    for (int v = 0; v < CPL; ++v) dk[v] = 0.0f;
#pragma unroll
                    for (int q = qa; q < qb; ++q)
#pragma unroll
                        for (int v = 0; v < CPL; ++v) {
                            acc[q][v] = fmaf(f[v], g[q][v], acc[q][v]);
                            dk[v] = fmaf(g[q][v], wy[q][v], dk[v]);
                        }
#pragma unroll
                    for (int v = 0; v < CPL; ++v) p = fmaf(dk[v], F[v], p);
                }
                pb[i] = p;
                // this warp is done with the slot; the producer refills it for edge e + RING_DEPTH once
                // every warp of the block has said so
                __syncwarp();
                if (lane == 0) ring_bar_arrive(ring.empty + slot);
                if (producer && eb + i + RING_DEPTH < e1) {
                    if (lane == 0) {
                        ring_bar_wait(ring.empty + slot, use & 1u);
                        ring_bulk_load(ring.rows + slot * (9 * C), GM + (size_t)j_ahead * (9 * C), ROW_BYTES,
                                       ring.full + slot);
                    }
                    if (eb + i + 1 + RING_DEPTH < e1) j_ahead = __ldg(ejk + eb + i + 1 + RING_DEPTH).x;
                }
            }
        }
#pragma unroll
        for (int o = 16, h = 4; h >= 1; o >>= 1, h >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < h; ++i) {
                const float send = up ? pb[i] : pb[i + h];
                const float keep = up ? pb[i + h] : pb[i];
                pb[i] = keep + __shfl_xor_sync(NNP_FULL_MASK, send, o);
            }
        }
        float tot = pb[0];
        tot += __shfl_xor_sync(NNP_FULL_MASK, tot, 2);
        tot += __shfl_xor_sync(NNP_FULL_MASK, tot, 1);
        const int idx = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
        if ((lane & 3) == 0 && eb + idx < e1 && __ldg(ejk + eb + idx).x != s) gd_slot[eb + idx] = tot;
    }
    float *out = GY + ((size_t)s * 9 + Q0) * C + cb;
#pragma unroll
    for (int q = 0; q < NQ; ++q) stv<CPL>(out + q * C, acc[q]);
}

// launched with exactly 64 * NPARTS threads: one receiver per block
template <int C, int CPL>
__global__ void __launch_bounds__(64 * (C / (32 * CPL)), 8 / (C / (32 * CPL))) k_edge_message_bwd_ring(TnDev d, int layer, const float *GM,
                                                                                  float *GY, float *gd_layer)
{
    NNP_PDL_SYNC();
    constexpr int NPARTS = C / (32 * CPL);
    __shared__ __align__(128) float rows[RING_DEPTH * 9 * C];
    __shared__ uint64_t bars[2 * RING_DEPTH];
    if (overflowed(d)) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s = blockIdx.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < RING_DEPTH; ++i) {
            ring_bar_init(bars + i, 1);                        // full: the producer's expect_tx arrival
            ring_bar_init(bars + RING_DEPTH + i, 2 * NPARTS);  // empty: one arrival per warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int part = warp >> 1, half = warp & 1;
    const int cb = part * 32 * CPL + lane * CPL;
    const float *tab = d.m.tables + (size_t)(layer + 1) * d.m.num_knots * 6 * C;
    float *gd_slot = gd_layer + (size_t)(2 * part + half) * d.capacity;
    RowRing<C> ring{rows, bars, bars + RING_DEPTH};
    if (half == 0) message_bwd_row_ring<C, CPL, 0, 2, 0, 4>(d, tab, GM, GY, d.Yc[layer], gd_slot, s, cb, ring, warp == 0);
    else message_bwd_row_ring<C, CPL, 2, 1, 4, 5>(d, tab, GM, GY, d.Yc[layer], gd_slot, s, cb, ring, false);
}

// Reverse of the edge op for the row of node a (the list is symmetric, so the scatter to senders
// is a gather over a's own row):
//   G_Y[a] += sum_e f_e[:,grp] * G_M[b]                         (b = sender of e)
//   slot e of this launch's g_d = sum_c sum_k <G_M[b], Yc[a]>_k * d f_e[c,k]/dd
// The second line is dE/dd of the REVERSE edge (a sends to b): the force kernel only ever uses
// g_d[e] + g_d[reverse(e)], which is symmetric, so storing the reverse edge's term in slot e is
// equivalent and needs no second gather (G_M[b] is already in registers, Yc[a] is the own node).
// Two edges are processed per iteration (loads of both in flight, one shared warp reduction).
// (launched with 128 threads: at 168 registers three blocks = 12 warps stay resident per SM)
template <int C, int CPL>
__global__ void __launch_bounds__(256) k_edge_message_bwd(TnDev d, int layer, const float *GM,
                                                          float *GY, float *gd_layer)
{
    NNP_PDL_SYNC();
    constexpr int NPARTS = C / (32 * CPL);
    if (overflowed(d)) return;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int s = gw / NPARTS, part = gw - s * NPARTS;
    if (s >= d.n) return;
    const int cb = part * 32 * CPL + lane * CPL;
    const float *tab = d.m.tables_mono + (size_t)(layer + 1) * (d.m.num_knots - 1) * 12 * C;
    float yown[9][CPL], acc[9][CPL];
    {
        const float *p = d.Yc[layer] + (size_t)s * 9 * C + cb;
        const float *py = GY + (size_t)s * 9 * C + cb;
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            ldv<CPL>(p + q * C, yown[q]);
            ldv<CPL>(py + q * C, acc[q]);
        }
    }
    const float inv_step = 1.0f / d.m.u_step;
    float *gd_slot = gd_layer + (size_t)part * d.capacity;   // this launch's own slots
    const int nk = d.m.num_knots;
    const int e0 = d.row_ptr[s], e1 = d.row_ptr[s + 1];
    for (int e = e0; e < e1; e += 2) {
        const bool two = e + 1 < e1;
        const int eb = two ? e + 1 : e;
        const int j0 = d.col[e], j1 = d.col[eb];
        float4 ga0 = d.geoA[e], ga1 = d.geoA[eb];
        const float u0 = d.geoB[e].w, u1 = d.geoB[eb].w;
        if (!two) ga1.y = ga1.z = 0.0f;          // the duplicated tail edge contributes nothing
        int kn0 = (int)ga0.x, kn1 = (int)ga1.x;
        kn0 = kn0 > nk - 2 ? nk - 2 : kn0;
        kn1 = kn1 > nk - 2 ? nk - 2 : kn1;
        const float t0 = ga0.x - (float)kn0, t1 = ga1.x - (float)kn1;
        const float su0 = -u0 * inv_step * ga0.y, su1 = -u1 * inv_step * ga1.y;
        const float *g0 = GM + (size_t)j0 * 9 * C + cb;
        const float *g1 = GM + (size_t)j1 * 9 * C + cb;
        float p0 = 0.0f, p1 = 0.0f;
        // the three component groups in turn, so only one group's radial values and one or two
        // gathered components are live at a time (registers -> occupancy)
        {   // I: component 0, metric 3
            float f0[CPL], df0[CPL], f1[CPL], df1[CPL], a[CPL], b[CPL];
            table_lookup_group<C, CPL>(tab, kn0, t0, cb, 0, f0, df0);
            table_lookup_group<C, CPL>(tab, kn1, t1, cb, 0, f1, df1);
            ldv<CPL>(g0, a);
            ldv<CPL>(g1, b);
#pragma unroll
            for (int v = 0; v < CPL; ++v) {
                acc[0][v] += (f0[v] * ga0.y) * a[v] + (f1[v] * ga1.y) * b[v];
                const float y3 = 3.0f * yown[0][v];
                p0 += a[v] * y3 * (df0[v] * su0 + f0[v] * ga0.z);
                p1 += b[v] * y3 * (df1[v] * su1 + f1[v] * ga1.z);
            }
        }
        {   // A: components 1..3, metric 2
            float f0[CPL], df0[CPL], f1[CPL], df1[CPL];
            table_lookup_group<C, CPL>(tab, kn0, t0, cb, 1, f0, df0);
            table_lookup_group<C, CPL>(tab, kn1, t1, cb, 1, f1, df1);
            float da[CPL], db[CPL];
#pragma unroll
            for (int v = 0; v < CPL; ++v) da[v] = db[v] = 0.0f;
#pragma unroll
            for (int q = 1; q < 4; ++q) {
                float a[CPL], b[CPL];
                ldv<CPL>(g0 + q * C, a);
                ldv<CPL>(g1 + q * C, b);
#pragma unroll
                for (int v = 0; v < CPL; ++v) {
                    acc[q][v] += (f0[v] * ga0.y) * a[v] + (f1[v] * ga1.y) * b[v];
                    da[v] += a[v] * yown[q][v];
                    db[v] += b[v] * yown[q][v];
                }
            }
#pragma unroll
            for (int v = 0; v < CPL; ++v) {
                p0 += 2.0f * da[v] * (df0[v] * su0 + f0[v] * ga0.z);
                p1 += 2.0f * db[v] * (df1[v] * su1 + f1[v] * ga1.z);
            }
        }
        {   // S: components 4..8; <a,y>_S = a4 y4 + a5 y5 + (a4+a5)(y4+y5) + 2 (a6 y6 + a7 y7 + a8 y8)
            float f0[CPL], df0[CPL], f1[CPL], df1[CPL];
            table_lookup_group<C, CPL>(tab, kn0, t0, cb, 2, f0, df0);
            table_lookup_group<C, CPL>(tab, kn1, t1, cb, 2, f1, df1);
            float da[CPL], db[CPL];
#pragma unroll
            for (int v = 0; v < CPL; ++v) da[v] = db[v] = 0.0f;
#pragma unroll
            for (int q = 4; q < 9; ++q) {
                float a[CPL], b[CPL];
                ldv<CPL>(g0 + q * C, a);
                ldv<CPL>(g1 + q * C, b);
#pragma unroll
                for (int v = 0; v < CPL; ++v) {
                    acc[q][v] += (f0[v] * ga0.y) * a[v] + (f1[v] * ga1.y) * b[v];
                    // weights of component q in the S inner product against the own node's Y
                    const float wy = q == 4 ? 2.0f * yown[4][v] + yown[5][v]
                                   : q == 5 ? 2.0f * yown[5][v] + yown[4][v]
                                            : 2.0f * yown[q][v];
                    da[v] += a[v] * wy;
                    db[v] += b[v] * wy;
                }
            }
#pragma unroll
            for (int v = 0; v < CPL; ++v) {
                p0 += da[v] * (df0[v] * su0 + f0[v] * ga0.z);
                p1 += db[v] * (df1[v] * su1 + f1[v] * ga1.z);
            }
        }
        // one butterfly for both edges: lanes 0-15 end with the sum of p0, lanes 16-31 with p1
        float x = (lane & 16) ? p1 : p0;
        const float y = (lane & 16) ? p0 : p1;
        x += __shfl_xor_sync(NNP_FULL_MASK, y, 16);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) x += __shfl_xor_sync(NNP_FULL_MASK, x, o);
        if (lane == 0 && j0 != s) gd_slot[e] = x;
        if (lane == 16 && two && j1 != s) gd_slot[e + 1] = x;
    }
    float *out = GY + (size_t)s * 9 * C + cb;
#pragma unroll
    for (int q = 0; q < 9; ++q) stv<CPL>(out + q * C, acc[q]);
}

// --------------------------------------------------------------------------------- readout
// feats = [|I|^2, |A|^2, |S|^2] -> LayerNorm_{3C}
template <int C>
__global__ void __launch_bounds__(256) k_readout_feats(TnDev d, const float *X)
{
    NNP_PDL_SYNC();
    constexpr int CPL = C / 32;
    const int lane = threadIdx.x & 31;
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= d.n) return;
    const int cb = lane * CPL;
    float x[9][CPL];
    const float *p = X + (size_t)s * 9 * C + cb;
#pragma unroll
    for (int q = 0; q < 9; ++q) ldv<CPL>(p + q * C, x[q]);
    float ft[3][CPL];
    float sum = 0.0f;
#pragma unroll
    for (int v = 0; v < CPL; ++v) {
        float c9[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) c9[q] = x[q][v];
        ft[0][v] = c9_dot_I(c9, c9);
        ft[1][v] = c9_dot_A(c9, c9);
        ft[2][v] = c9_dot_S(c9, c9);
        sum += ft[0][v] + ft[1][v] + ft[2][v];
    }
    const float mean = nnp_warp_sum(sum) * (1.0f / (3 * C));
    float var = 0.0f;
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int v = 0; v < CPL; ++v) var += (ft[k][v] - mean) * (ft[k][v] - mean);
    var = nnp_warp_sum(var) * (1.0f / (3 * C));
    const float rstd = rsqrtf(var + LN_EPS);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float g[CPL], bb[CPL], out[CPL];
        ldv<CPL>(d.m.out_norm_g + k * C + cb, g);
        ldv<CPL>(d.m.out_norm_b + k * C + cb, bb);
#pragma unroll
        for (int v = 0; v < CPL; ++v) out[v] = (ft[k][v] - mean) * rstd * g[v] + bb[v];
        stv<CPL>(d.lnr + (size_t)s * 3 * C + k * C + cb, out);
    }
}

// per-atom energy: (silu(r1) . h2_w + h2_b) * std + mean  (graphnet.py:403-406), original order;
// also the head's own reverse (g_r1) and the caller's per-atom copy
__global__ void k_head(TnDev d, int H)
{
    NNP_PDL_SYNC();
    const int lane = threadIdx.x & 31;
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= d.n) return;
    float part = 0.0f;
    for (int h = lane; h < H; h += 32) {
        const float r = d.r1[(size_t)s * H + h], w = d.m.h2_w[h];
        part += nnp_silu(r) * w;
        // reverse of this very line: dE/dr1 = std * h2_w * silu'(r1)  (energy-only calls ignore it)
        d.g_r1[(size_t)s * H + h] = d.m.std * w * nnp_silu_grad(r);
    }
    part = nnp_warp_sum(part);
    if (lane == 0) {
        const float e = (part + d.m.h2_b) * d.m.std + d.m.mean;
        const int i = d.order ? d.order[s] : s;
        d.e_atom[i] = e;
        if (d.per_atom) d.per_atom[i] = e;
    }
}

// per-sample sums in float64, fixed order (graphnet.py:411 segment_sum over batch)
__global__ void __launch_bounds__(1024) k_energy_sum(TnDev d)
{
    NNP_PDL_SYNC();
    const int b = blockIdx.x;
    const int p0 = d.sample_ptr[b], p1 = d.sample_ptr[b + 1];
    double acc = 0.0;
    for (int i = p0 + threadIdx.x; i < p1; i += blockDim.x) acc += (double)d.e_atom[i];
    __shared__ double sh[32];
    acc = nnp_warp_sum(acc);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
        d.energy[b] = (float)t;
    }
}

// reverse of k_readout_feats: GX = 2 * g_feats[grp] * X_part
template <int C>
__global__ void __launch_bounds__(256) k_readout_bwd(TnDev d, const float *X, float *GX, const float *Dc_last,
                                                     float *GD)
{
    NNP_PDL_SYNC();
    constexpr int CPL = C / 32;
    const int lane = threadIdx.x & 31;
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= d.n) return;
    const int cb = lane * CPL;
    float x[9][CPL];
    const float *p = X + (size_t)s * 9 * C + cb;
#pragma unroll
    for (int q = 0; q < 9; ++q) ldv<CPL>(p + q * C, x[q]);
    float ft[3][CPL];
    float sum = 0.0f;
#pragma unroll
    for (int v = 0; v < CPL; ++v) {
        float c9[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) c9[q] = x[q][v];
        ft[0][v] = c9_dot_I(c9, c9);
        ft[1][v] = c9_dot_A(c9, c9);
        ft[2][v] = c9_dot_S(c9, c9);
        sum += ft[0][v] + ft[1][v] + ft[2][v];
    }
    const float inv_n = 1.0f / (3 * C);
    const float mean = nnp_warp_sum(sum) * inv_n;
    float var = 0.0f;
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int v = 0; v < CPL; ++v) var += (ft[k][v] - mean) * (ft[k][v] - mean);
    var = nnp_warp_sum(var) * inv_n;
    const float rstd = rsqrtf(var + LN_EPS);
    float gxh[3][CPL], xh[3][CPL];
    float s1 = 0.0f, s2 = 0.0f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float g[CPL], gy[CPL];
        ldv<CPL>(d.m.out_norm_g + k * C + cb, g);
        ldv<CPL>(d.g_lnr + (size_t)s * 3 * C + k * C + cb, gy);
#pragma unroll
        for (int v = 0; v < CPL; ++v) {
            xh[k][v] = (ft[k][v] - mean) * rstd;
            gxh[k][v] = gy[v] * g[v];
            s1 += gxh[k][v];
            s2 += gxh[k][v] * xh[k][v];
        }
    }
    s1 = nnp_warp_sum(s1) * inv_n;
    s2 = nnp_warp_sum(s2) * inv_n;
    float *out = GX + (size_t)s * 9 * C + cb;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        const int k = group_of(q);
#pragma unroll
        for (int v = 0; v < CPL; ++v) {
            const float gf = rstd * (gxh[k][v] - s1 - xh[k][v] * s2);
            x[q][v] = 2.0f * gf * x[q][v];          // x now holds GX
        }
        stv<CPL>(out + q * C, x[q]);
    }
    if (!Dc_last) return;
    // fused k_residual_bwd of the last layer: G_D = GX + GX*D^T + D^T*GX
    const float *pd = Dc_last + (size_t)s * 9 * C + cb;
    float *og = GD + (size_t)s * 9 * C + cb;
    float dcv[9][CPL];
#pragma unroll
    for (int q = 0; q < 9; ++q) ldv<CPL>(pd + q * C, dcv[q]);
#pragma unroll
    for (int v = 0; v < CPL; ++v) {
        float g9[9], d9[9], gd9[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            g9[q] = x[q][v];
            d9[q] = dcv[q][v];
        }
        residual_bwd(g9, d9, gd9);
#pragma unroll
        for (int q = 0; q < 9; ++q) dcv[q][v] = gd9[q];
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) stv<CPL>(og + q * C, dcv[q]);
}

// G_X0 = G_X0part + 2 * g_n0 * X0, g_n0 = LayerNorm_C backward of g_ln0
template <int C>
__global__ void __launch_bounds__(256) k_embed_norm_bwd(TnDev d, float *GX0)
{
    NNP_PDL_SYNC();
    constexpr int CPL = C / 32;
    const int lane = threadIdx.x & 31;
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= d.n) return;
    const int cb = lane * CPL;
    float nrm[CPL], g[CPL], gy[CPL];
    ldv<CPL>(d.n0 + (size_t)s * C + cb, nrm);
    ldv<CPL>(d.m.init_norm_g + cb, g);
    ldv<CPL>(d.g_ln0 + (size_t)s * C + cb, gy);
    float sum = 0.0f;
#pragma unroll
    for (int v = 0; v < CPL; ++v) sum += nrm[v];
    const float mean = nnp_warp_sum(sum) * (1.0f / C);
    float var = 0.0f;
#pragma unroll
    for (int v = 0; v < CPL; ++v) var += (nrm[v] - mean) * (nrm[v] - mean);
    var = nnp_warp_sum(var) * (1.0f / C);
    const float rstd = rsqrtf(var + LN_EPS);
    float xh[CPL], gxh[CPL];
    float s1 = 0.0f, s2 = 0.0f;
#pragma unroll
    for (int v = 0; v < CPL; ++v) {
        xh[v] = (nrm[v] - mean) * rstd;
        gxh[v] = gy[v] * g[v];
        s1 += gxh[v];
        s2 += gxh[v] * xh[v];
    }
    s1 = nnp_warp_sum(s1) * (1.0f / C);
    s2 = nnp_warp_sum(s2) * (1.0f / C);
    float gn[CPL];
#pragma unroll
    for (int v = 0; v < CPL; ++v) gn[v] = rstd * (gxh[v] - s1 - xh[v] * s2);
    const float *x0 = d.X0 + (size_t)s * 9 * C + cb;
    float *out = GX0 + (size_t)s * 9 * C + cb;
    float t[9][CPL];
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        float x[CPL];
        ldv<CPL>(x0 + q * C, x);
        ldv<CPL>(out + q * C, t[q]);
#pragma unroll
        for (int v = 0; v < CPL; ++v) t[q][v] += 2.0f * gn[v] * x[v];
        stv<CPL>(out + q * C, t[q]);
    }
    if (!d.Hb) return;
    // bias column of the projected embedding reverse:
    //   Hb[s][slot][q] = sum_c (z_recv[z_s][c] + z_send[species(slot)][c]) dp_b[grp(q)][c] G[q][c]
    float zr[CPL], part[EMB_SLOTS * 9];
    ldv<CPL>(d.m.z_recv + (size_t)d.zs[s] * C + cb, zr);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float b[CPL];
        ldv<CPL>(d.m.dp_b + k * C + cb, b);
#pragma unroll
        for (int q = (k == 0 ? 0 : (k == 1 ? 1 : 4)); q < (k == 0 ? 1 : (k == 1 ? 4 : 9)); ++q)
#pragma unroll
            for (int v = 0; v < CPL; ++v) t[q][v] *= b[v];
    }
#pragma unroll
    for (int sl = 0; sl < EMB_SLOTS; ++sl) {
        const int z = d.slot_species[sl];
        float zz[CPL];
        ldv<CPL>(d.m.z_send + (size_t)(z < 0 ? 0 : z) * C + cb, zz);
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            float a = 0.0f;
#pragma unroll
            for (int v = 0; v < CPL; ++v) a = fmaf(zr[v] + zz[v], t[q][v], a);
            part[sl * 9 + q] = a;
        }
    }
    // 36 warp sums: the first 32 by a transposing butterfly (31 shuffles; lane l ends up with the
    // total of value l), the last four one by one
    float tail[EMB_SLOTS * 9 - 32];
#pragma unroll
    for (int i = 32; i < EMB_SLOTS * 9; ++i) tail[i - 32] = nnp_warp_sum(part[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const float send = up ? part[i] : part[i + o];
            const float keep = up ? part[i + o] : part[i];
            part[i] = keep + __shfl_xor_sync(NNP_FULL_MASK, send, o);
        }
    }
    float *hb = d.Hb + (size_t)s * (EMB_SLOTS * 9);
    hb[lane] = part[0];
#pragma unroll
    for (int i = 32; i < EMB_SLOTS * 9; ++i)
        if (lane == i - 32) hb[i] = tail[i - 32];
}

// reverse of k_embed_edge: per edge g_d += dE/dd (through dp(rho) and phi) and g_u = dE/du
template <int C, int CPL>
__global__ void __launch_bounds__(256) k_embed_edge_bwd(TnDev d, const float *GX0)
{
    NNP_PDL_SYNC();
    constexpr int NPARTS = C / (32 * CPL);
    if (overflowed(d)) return;
    if (d.embed_fast && d.embed_fast[0]) return;   // the projected kernels do this step's embedding reverse
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int s = gw / NPARTS, part = gw - s * NPARTS;
    if (s >= d.n) return;
    const int cb = part * 32 * CPL + lane * CPL;
    float zr[CPL];
    ldv<CPL>(d.m.z_recv + (size_t)d.zs[s] * C + cb, zr);
    float G[9][CPL], g0x3[CPL], szz[CPL];
    const float *p = GX0 + (size_t)s * 9 * C + cb;
#pragma unroll
    for (int q = 0; q < 9; ++q) ldv<CPL>(p + q * C, G[q]);
#pragma unroll
    for (int v = 0; v < CPL; ++v) {
        g0x3[v] = 3.0f * G[0][v];
        szz[v] = -G[4][v] - G[5][v];
    }
    const float inv_step = 1.0f / d.m.u_step;
    const int e0 = d.row_ptr[s], e1 = d.row_ptr[s + 1];
    // next edge's scalars are fetched one iteration ahead (their latency was the top stall)
    int nj = 0, nz = 0;
    float4 nga = make_float4(0.f, 0.f, 0.f, 0.f), ngb = nga;
    if (e0 < e1) {
        nj = d.col[e0];
        nz = d.zs[nj];
        nga = d.geoA[e0];
        ngb = d.geoB[e0];
    }
    float kd = 0.0f;
    float4 ku = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int e = e0; e < e1; ++e) {
        const int zj = nz;
        const float4 ga = nga, gb = ngb;
        if (e + 1 < e1) {
            nj = d.col[e + 1];
            nz = d.zs[nj];
            nga = d.geoA[e + 1];
            ngb = d.geoB[e + 1];
        }
        // (a self loop has no geometry: its zero envelope derivative and unit vector make every
        //  term below vanish, and the flush skips its slot)
        float zsnd[CPL];
        ldv<CPL>(d.m.z_send + (size_t)zj * C + cb, zsnd);
        float f[3][CPL], df[3][CPL];
        table_lookup<C, CPL, true>(d.m.tables_mono, d.m.num_knots, ga.x, cb, f, df);
        // per-edge scalars of the unit tensors: <G, b>_A = 2 (G1 ux + G2 uy + G3 uz),
        // <G, b>_S = G4 (2 b4 + b5) + G5 (2 b5 + b4) + 2 (G6 b6 + G7 b7 + G8 b8)
        const float uu = (gb.x * gb.x + gb.y * gb.y + gb.z * gb.z) * (1.0f / 3.0f);
        const float b4 = gb.x * gb.x - uu, b5 = gb.y * gb.y - uu;
        const float a1 = 2.0f * gb.x, a2 = 2.0f * gb.y, a3 = 2.0f * gb.z;
        const float s4 = 2.0f * b4 + b5, s5 = 2.0f * b5 + b4;
        const float s6 = a1 * gb.y, s7 = a1 * gb.z, s8 = a2 * gb.z;
        const float su = -gb.w * inv_step * ga.y;
        float pd = 0.0f, px = 0.0f, py = 0.0f, pz = 0.0f;
#pragma unroll
        for (int v = 0; v < CPL; ++v) {
            const float Z = zr[v] + zsnd[v];
            const float gA = fmaf(G[1][v], a1, fmaf(G[2][v], a2, G[3][v] * a3));
            const float gS = fmaf(G[4][v], s4, fmaf(G[5][v], s5, fmaf(G[6][v], s6, fmaf(G[7][v], s7, G[8][v] * s8))));
            const float F0 = fmaf(df[0][v], su, f[0][v] * ga.z);
            const float F1 = fmaf(df[1][v], su, f[1][v] * ga.z);
            const float F2 = fmaf(df[2][v], su, f[2][v] * ga.z);
            pd = fmaf(Z, fmaf(g0x3[v], F0, fmaf(gA, F1, gS * F2)), pd);
            const float Zp = Z * ga.y;
            const float w1 = f[1][v] * Zp, w2 = f[2][v] * Zp;
            const float vx = fmaf(G[4][v], gb.x, fmaf(G[6][v], gb.y, G[7][v] * gb.z));
            const float vy = fmaf(G[6][v], gb.x, fmaf(G[5][v], gb.y, G[8][v] * gb.z));
            const float vz = fmaf(G[7][v], gb.x, fmaf(G[8][v], gb.y, szz[v] * gb.z));
            px = fmaf(w1, G[1][v], fmaf(w2, vx, px));
            py = fmaf(w1, G[2][v], fmaf(w2, vy, py));
            pz = fmaf(w1, G[3][v], fmaf(w2, vz, pz));
        }
        {   // four warp sums with 6 + 4 shuffles instead of 20: transpose-reduce, then broadcast
            float a = (lane & 16) ? px : pd, b = (lane & 16) ? pd : px;
            a += __shfl_xor_sync(NNP_FULL_MASK, b, 16);
            float c = (lane & 16) ? pz : py, f2 = (lane & 16) ? py : pz;
            c += __shfl_xor_sync(NNP_FULL_MASK, f2, 16);
            float x = (lane & 8) ? c : a;
            const float y = (lane & 8) ? a : c;
            x += __shfl_xor_sync(NNP_FULL_MASK, y, 8);
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) x += __shfl_xor_sync(NNP_FULL_MASK, x, o);
            pd = __shfl_sync(NNP_FULL_MASK, x, 0);
            px = __shfl_sync(NNP_FULL_MASK, x, 16);
            py = __shfl_sync(NNP_FULL_MASK, x, 8);
            pz = __shfl_sync(NNP_FULL_MASK, x, 24);
        }
        // every lane holds the four totals; lane (e - e0) % 32 keeps them, and a full group of 32
        // edges is written with one coalesced store instead of 32 single-lane ones
        if (lane == ((e - e0) & 31)) {
            kd = pd;
            ku = make_float4(2.0f * px, 2.0f * py, 2.0f * pz, 0.0f);
        }
        if (((e - e0) & 31) == 31 || e + 1 == e1) {
            const int eb = e0 + ((e - e0) & ~31) + lane;      // this lane's edge of the group
            if (eb <= e && d.col[eb] != s) {
                d.g_d[(size_t)part * d.capacity + eb] = kd;      // slot 0 .. nparts-1: the embedding's
                d.g_u[(size_t)part * d.capacity + eb] = ku;
            }
        }
    }
}

// Reverse of k_embed_edge through the node-level projection.  Hs[i][q][slot*32+k] and
// Hr[i][q][slot*32+k] are dE/dX0 contracted over channels against z_send[species(slot)] * dp_w and
// z_recv[species(slot)] * dp_w (two channel-mix shaped GEMMs); with
//   Hc[slot][q][k] = Hs[i][q][slot][k] + Hr[i][q][slot(z_i)][k],   chi_k = phi rho_k,   psi_k = d(phi rho_k)/dd
// an edge e = (i <- j), slot = slot(z_j), gives
//   dE/dd_e = sum_k psi_k (3 Hc[0] + sum_{q in A} 2 u_q Hc[q] + sum_{q in S} s_q Hc[q])[k]
//   dE/du_e = 2 sum_k chi_k (Hc[1..3] + sym(Hc[4..8]) u)[k]
// plus the bias column (chi = phi, psi = phi') from Hb.  One warp per receiver stages Hc in shared
// memory, then every lane owns one edge of the row: no reductions, coalesced stores.
// rho_k = exp(-beta_k (u - mu_k)^2), u = exp(cutoff_lower - d)  (radial.py:53-59).
constexpr int EMB_PROJ_WARPS = 4;
constexpr int EMB_PROJ_STRIDE = 9 * EMB_K + 4;   // slot stride: slots land on different banks
__global__ void __launch_bounds__(EMB_PROJ_WARPS * 32) k_embed_edge_bwd_proj(TnDev d, const float *Hs,
                                                                             const float *Hr)
{
    NNP_PDL_SYNC();
    __shared__ __align__(16) float hc_all[EMB_PROJ_WARPS][EMB_SLOTS * EMB_PROJ_STRIDE];
    __shared__ __align__(16) float hb_all[EMB_PROJ_WARPS][EMB_SLOTS * 9 + 4];
    __shared__ __align__(16) float mu_s[EMB_K], beta_s[EMB_K];
    if (threadIdx.x < EMB_K) {
        mu_s[threadIdx.x] = d.m.rbf_means[threadIdx.x];
        beta_s[threadIdx.x] = d.m.rbf_betas[threadIdx.x];
    }
    __syncthreads();
    if (overflowed(d) || !d.embed_fast[0]) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s = blockIdx.x * EMB_PROJ_WARPS + warp;
    if (s >= d.n) return;
    float *hc = hc_all[warp], *hb = hb_all[warp];
    {
        const int my = d.slot_of_z[d.zs[s]];
        const float *ps = Hs + (size_t)s * 9 * (EMB_SLOTS * EMB_K) + lane;
        const float *pr = Hr + (size_t)s * 9 * (EMB_SLOTS * EMB_K) + my * EMB_K + lane;
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            const float r = pr[q * (EMB_SLOTS * EMB_K)];
#pragma unroll
            for (int sl = 0; sl < EMB_SLOTS; ++sl)
                hc[sl * EMB_PROJ_STRIDE + q * EMB_K + lane] = ps[q * (EMB_SLOTS * EMB_K) + sl * EMB_K] + r;
        }
        const float *pb = d.Hb + (size_t)s * (EMB_SLOTS * 9);
        hb[lane] = pb[lane];
        if (lane < EMB_SLOTS * 9 - 32) hb[32 + lane] = pb[32 + lane];
    }
    __syncwarp();
    const int e0 = d.row_ptr[s], e1 = d.row_ptr[s + 1];
    for (int e = e0 + lane; e < e1; e += 32) {
        const int j = d.col[e];
        if (j == s) continue;                       // a self loop has no geometry
        const int sl = d.slot_of_z[d.zs[j]];
        const float4 ga = d.geoA[e];
        const float4 gb = d.geoB[e];
        const float u = gb.w, phi = ga.y, dphi = ga.z;
        const float c1 = 2.0f * u * phi;            // psi_k = rho_k (c1 beta_k (u - mu_k) + phi')
        float hp[9], hx[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) hp[q] = hx[q] = 0.0f;
        const float4 *H4 = reinterpret_cast<const float4 *>(hc + sl * EMB_PROJ_STRIDE);
#pragma unroll 2
        for (int k4 = 0; k4 < EMB_K / 4; ++k4) {
            const float4 mu = reinterpret_cast<const float4 *>(mu_s)[k4];
            const float4 be = reinterpret_cast<const float4 *>(beta_s)[k4];
            float chi[4], psi[4];
            {
                const float m4[4] = {mu.x, mu.y, mu.z, mu.w}, b4[4] = {be.x, be.y, be.z, be.w};
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const float df = u - m4[v];
                    const float t = b4[v] * df;
                    const float rho = __expf(-t * df);
                    chi[v] = rho * phi;
                    psi[v] = rho * fmaf(c1, t, dphi);
                }
            }
#pragma unroll
            for (int q = 0; q < 9; ++q) {
                const float4 h = H4[q * (EMB_K / 4) + k4];
                hp[q] = fmaf(psi[0], h.x, fmaf(psi[1], h.y, fmaf(psi[2], h.z, fmaf(psi[3], h.w, hp[q]))));
                if (q > 0)
                    hx[q] = fmaf(chi[0], h.x, fmaf(chi[1], h.y, fmaf(chi[2], h.z, fmaf(chi[3], h.w, hx[q]))));
            }
        }
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            const float b = hb[sl * 9 + q];
            hp[q] = fmaf(dphi, b, hp[q]);
            hx[q] = fmaf(phi, b, hx[q]);
        }
        const float uu = (gb.x * gb.x + gb.y * gb.y + gb.z * gb.z) * (1.0f / 3.0f);
        const float b4 = gb.x * gb.x - uu, b5 = gb.y * gb.y - uu;
        const float a1 = 2.0f * gb.x, a2 = 2.0f * gb.y, a3 = 2.0f * gb.z;
        const float pd = 3.0f * hp[0] + a1 * hp[1] + a2 * hp[2] + a3 * hp[3] + (2.0f * b4 + b5) * hp[4] +
                         (2.0f * b5 + b4) * hp[5] + a1 * gb.y * hp[6] + a1 * gb.z * hp[7] + a2 * gb.z * hp[8];
        const float px = hx[1] + hx[4] * gb.x + hx[6] * gb.y + hx[7] * gb.z;
        const float py = hx[2] + hx[6] * gb.x + hx[5] * gb.y + hx[8] * gb.z;
        const float pz = hx[3] + hx[7] * gb.x + hx[8] * gb.y - (hx[4] + hx[5]) * gb.z;
        d.g_d[e] = pd;                              // slot 0 of the embedding's share
        d.g_u[e] = make_float4(2.0f * px, 2.0f * py, 2.0f * pz, 0.0f);
    }
}

// forces: F_i = -sum_{e in row i} [ (g_d[e] + g_d[e']) u_e + (1 - u u^T)(g_u[e] - g_u[e']) / d_e ]
// with e' the reverse edge (u_e' = -u_e), precomputed by k_edge_rev.  One warp per atom: lanes
// take the row's edges 32 at a time (every edge costs a few dependent scattered reads), then a
// fixed-order butterfly sums the three components, so the result is reproducible.
__global__ void __launch_bounds__(256) k_forces(TnDev d)
{
    NNP_PDL_SYNC();
    if (overflowed(d)) return;
    const int lane = threadIdx.x & 31;
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= d.n) return;
    float gx = 0.0f, gy = 0.0f, gz = 0.0f;
    const int e0 = d.row_ptr[s], e1 = d.row_ptr[s + 1];
    for (int e = e0 + lane; e < e1; e += 32) {
        const int j = d.col[e];
        if (j == s) continue;
        const int er = d.rev[e];
        const float4 ga = d.geoA[e];
        const float4 gb = d.geoB[e];
        float gd = 0.0f, vx = 0.0f, vy = 0.0f, vz = 0.0f;
        for (int p = 0; p < d.nparts; ++p) {
            const size_t po = (size_t)p * d.capacity;
            const float4 ue = d.g_u[po + e], ur = d.g_u[po + er];
            vx += ue.x - ur.x;
            vy += ue.y - ur.y;
            vz += ue.z - ur.z;
        }
        for (int p = 0; p < d.gd_slots * (d.m.num_layers + 1); ++p) {
            const size_t po = (size_t)p * d.capacity;
            gd += d.g_d[po + e] + d.g_d[po + er];
        }
        const float dot = vx * gb.x + vy * gb.y + vz * gb.z;
        gx += gd * gb.x + (vx - gb.x * dot) * ga.w;
        gy += gd * gb.y + (vy - gb.y * dot) * ga.w;
        gz += gd * gb.z + (vz - gb.z * dot) * ga.w;
    }
    gx = nnp_warp_sum(gx);
    gy = nnp_warp_sum(gy);
    gz = nnp_warp_sum(gz);
    if (lane == 0) {
        const size_t o = 3 * (size_t)(d.order ? d.order[s] : s);
        d.forces[o] = -gx;
        d.forces[o + 1] = -gy;
        d.forces[o + 2] = -gz;
    }
}

// --------------------------------------------------------------------------------- host side
size_t carve(TnDev &d, void *ws)
{
    NnpArena ar(ws);
    const size_t n = (size_t)d.n, C = (size_t)d.m.channels, cap = (size_t)d.capacity;
    const size_t T = n * 9 * C;
    const int L = d.m.num_layers;
    d.col = ar.take<int>(cap);
    d.rev = ar.take<int>(cap);
    d.newpos = ar.take<int>(cap);
    d.geoA = ar.take<float4>(cap);
    d.geoB = ar.take<float4>(cap);
    d.ejk = ar.take<int2>(cap);
    d.hwV = ar.take<float4>(cap);
    d.hwD = ar.take<float4>(cap);
    d.ezs = ar.take<int>(cap);
    d.g_d = ar.take<float>(cap * NNP_GD_SLOTS * (size_t)(L + 1));
    d.g_u = ar.take<float4>(cap * NNP_PARTS);
    d.zs = ar.take<int>(n);
    d.sample_ptr = ar.take<int>((size_t)d.n_samples + 1);
    d.X0 = ar.take<float>(T);
    d.n0 = ar.take<float>(n * C);
    d.ln0 = ar.take<float>(n * C);
    d.e0 = ar.take<float>(n * 2 * C);
    d.se0 = ar.take<float>(n * 2 * C);
    d.e1 = ar.take<float>(n * 3 * C);
    d.Xm = ar.take<float>(T);
    d.Xa = ar.take<float>(T);
    d.Xb = ar.take<float>(T);
    for (int l = 0; l < L; ++l) {
        d.Xh[l] = ar.take<float>(T);
        d.nx[l] = ar.take<float>(n * C);
        d.Yc[l] = ar.take<float>(T);
        d.Mc[l] = ar.take<float>(T);
        d.Dc[l] = ar.take<float>(T);
    }
    d.Qc = ar.take<float>(T);
    d.lnr = ar.take<float>(n * 3 * C);
    d.r0 = ar.take<float>(n * C);
    d.sr0 = ar.take<float>(n * C);
    d.r1 = ar.take<float>(n * (C / 2));
    d.e_atom = ar.take<float>(n);
    d.G1 = ar.take<float>(T);
    d.G2 = ar.take<float>(T);
    d.G3 = ar.take<float>(T);
    d.g_r1 = ar.take<float>(n * (C / 2));
    d.g_r0 = ar.take<float>(n * C);
    d.g_lnr = ar.take<float>(n * 3 * C);
    d.g_e1 = ar.take<float>(n * 3 * C);
    d.g_e0 = ar.take<float>(n * 2 * C);
    d.g_ln0 = ar.take<float>(n * C);
    if (d.m.embed_projection) {
        d.present = ar.take<int>((size_t)d.m.max_z);
        d.slot_of_z = ar.take<int>((size_t)d.m.max_z);
        d.slot_species = ar.take<int>(EMB_SLOTS);
        d.embed_fast = ar.take<int>(1);
        d.Wproj = ar.take<float>((size_t)3 * 2 * EMB_SLOTS * EMB_K * C);
        d.Hb = ar.take<float>(n * EMB_SLOTS * 9);
    }
    return ar.bytes();
}

int validate_model(const nnp_tn_model *m)
{
    NNP_CHECK_ARG(m != nullptr, "model is NULL");
    NNP_CHECK_ARG(m->channels == 32 || m->channels == 64 || m->channels == 128,
                  "channels must be 32, 64 or 128");
    NNP_CHECK_ARG(m->num_layers >= 0 && m->num_layers <= NNP_TN_MAX_LAYERS, "num_layers out of range");
    NNP_CHECK_ARG(m->num_knots >= 2, "num_knots must be >= 2");
    NNP_CHECK_ARG(m->gemm_mode == 0 || m->gemm_mode == 1 || m->gemm_mode == 3 || m->gemm_mode == 5 || m->gemm_mode == 8,
                  "gemm_mode must be 0 (default), 1, 3, 5 or 8");
    NNP_CHECK_ARG(m->u_step > 0.0f, "u_step must be positive");
    NNP_CHECK_ARG(m->cutoff_lower >= 0.0f && m->cutoff_lower < m->cutoff_upper, "bad cutoffs");
    NNP_CHECK_ARG(!m->embed_projection || (m->num_rbf == EMB_K && m->channels == EMB_SLOTS * EMB_K && m->dp_wT && m->dp_b && m->rbf_means &&
                                           m->rbf_betas && m->max_z >= 1),
                  "embed_projection needs num_rbf == 32, 128 channels and the dp / rbf arrays");
    return NNP_OK;
}

GemmArgs plain_gemm(const float *A, const nnp_gemm_weight &W, const float *bias, float *out, int M,
                    int N, int K, const float *aux = nullptr, int ldaux = 0)
{
    GemmArgs g{};
    g.A = A;
    g.W = W.w;
    g.bias = bias;
    g.out = out;
    g.aux = aux;
    g.M = M;
    g.N = N;
    g.K = K;
    g.lda = K;
    g.ldo = N;
    g.ldaux = ldaux;
    return g;
}

// the three component groups (I: 1 comp, A: 3, S: 5) of a [N,9,C] tensor against W[3][C][C]
GemmBatch mix_gemm(const float *A, const nnp_gemm_weight *W3, float *out, int n, int C,
                   float *out2 = nullptr, const float *aux = nullptr, int ldaux = 0)
{
    static const int ncomp[3] = {1, 3, 5}, q0[3] = {0, 1, 4};
    GemmBatch b{};
    for (int k = 0; k < 3; ++k) {
        GemmArgs &g = b.g[k];
        g.A = A;
        g.W = W3[k].w;
        g.out = out;
        g.out2 = out2;
        g.aux = aux;
        g.M = n * ncomp[k];
        g.N = C;
        g.K = C;
        g.lda = C;
        g.ldo = C;
        g.ldaux = ldaux;
        g.ncomp = ncomp[k];
        g.q0 = q0[k];
        g.grp = k;
    }
    return b;
}

// Channels per lane of the four row-walking edge kernels (1, 2 or 4; C / (32 * CPL) warps share a
// node's row).  Fewer channels per lane = fewer registers and more warps in flight; tunable
// through NNP_CPL_{EMB,FWD,BWD,EMBBWD} for measurements.
struct EdgeTuning {
    int emb, fwd, bwd, embbwd, bwd_block, fwd_block, emb_block, bwd_split, emb_split;
};
static int env_int(const char *name, int fallback)
{
    const char *v = getenv(name);
    return v ? atoi(v) : fallback;
}
static const EdgeTuning &edge_tuning()
{
    static const EdgeTuning t = {env_int("NNP_CPL_EMB", 4), env_int("NNP_CPL_FWD", 4),
                                 env_int("NNP_CPL_BWD", 4), env_int("NNP_CPL_EMBBWD", 4),
                                 std::min(env_int("NNP_BWD_BLOCK", 128), 128), std::min(env_int("NNP_FWD_BLOCK", 64), 128), env_int("NNP_EMB_BLOCK", 128),
                                 env_int("NNP_BWD_SPLIT", 1),   // 1 = register gather, two warps per receiver (default); 2 = bulk-copy ring
                                                                // (measured slower: 2.15 vs 1.30 ms per step); 0 = one warp per part, monomial tables
                                 env_int("NNP_EMB_SPLIT", 2)};  // knot-cached embedding edge kernels: 2 = two warps per receiver up to 2 048 atoms, one warp
                                                                // beyond (default); 1 / 3 = always two / one; 0 = the round-1 kernels on monomial tables
    return t;
}
#define EDGE_DISPATCH(C, cpl_req, LAUNCH)                         \
    do {                                                          \
        int cpl__ = (cpl_req);                                    \
        if (cpl__ * 32 > (C)) cpl__ = (C) / 32;                   \
        if (cpl__ != 1 && cpl__ != 2 && cpl__ != 4) cpl__ = 1;    \
        if (cpl__ == 4) {                                         \
            if constexpr ((C) >= 128) { constexpr int CPL = 4; LAUNCH; } \
        } else if (cpl__ == 2) {                                  \
            if constexpr ((C) >= 64) { constexpr int CPL = 2; LAUNCH; }  \
        } else {                                                  \
            constexpr int CPL = 1; LAUNCH;                        \
        }                                                         \
    } while (0)

template <int C>
int run_step(TnDev &d, cudaStream_t st)
{
    const int n = d.n, L = d.m.num_layers, H = C / 2;
    const int warp_blocks = nnp_blocks(n, 8);
    const int ew_blocks = nnp_blocks((int64_t)n * C, 256);
    const nnp_tn_model &m = d.m;
    const EdgeTuning &tune = edge_tuning();
    {
        auto parts = [](int cpl) {
            if (cpl * 32 > C) cpl = C / 32;
            if (cpl != 1 && cpl != 2 && cpl != 4) cpl = 1;
            return C / (32 * cpl);
        };
        d.nparts = std::max(parts(tune.bwd), parts(tune.embbwd));
        d.gd_slots = std::max(parts(tune.embbwd), (tune.bwd_split ? 2 : 1) * parts(tune.bwd));
    }
    int rc;
#define RUN(x)            \
    do {                  \
        rc = (x);         \
        if (rc) return rc; \
    } while (0)

    { NNP_PROF("k_prep_nodes", st); nnp_launch((k_prep_nodes), NNP_GRID(nnp_blocks(n, 256)), 256, 0, st, d); }
    { NNP_PROF("k_edge_order", st); nnp_launch((k_edge_order), NNP_GRID(warp_blocks), 256, 0, st, d); }
    { NNP_PROF("k_edge_rev", st); nnp_launch((k_edge_rev), NNP_GRID(nnp_blocks(d.capacity, 256)), 256, 0, st, d); }
    if (d.m.embed_projection && d.forces) { NNP_PROF("k_embed_slots", st); nnp_launch((k_embed_slots), NNP_GRID(3 * 2 * EMB_SLOTS), 256, 0, st, d); }

    // ---- embedding
    // two knot-cached warps per receiver pay off for small systems only (measured: 22 atoms 14.2 vs
    // 21.6 us; config C 0.343 vs 0.338 ms; config D 1.01 vs 0.88 ms): NNP_EMB_SPLIT = 2 picks by size
    if (tune.emb_split == 3 || (tune.emb_split == 2 && n > 2048)) { NNP_PROF("k_embed_edge", st); EDGE_DISPATCH(C, tune.emb, (nnp_launch((k_embed_edge_knots<C, CPL>), NNP_GRID(nnp_blocks((int64_t)n * (C / (32 * CPL)), 2)), 64, 0, st, d))); }
    else if (tune.emb_split == 1 || (tune.emb_split == 2 && n <= 2048)) { NNP_PROF("k_embed_edge", st); EDGE_DISPATCH(C, tune.emb, (nnp_launch((k_embed_edge_split<C, CPL>), NNP_GRID(nnp_blocks((int64_t)n * 2 * (C / (32 * CPL)), 2)), 64, 0, st, d))); }
    else { NNP_PROF("k_embed_edge", st); EDGE_DISPATCH(C, tune.emb, (nnp_launch((k_embed_edge<C, CPL>), NNP_GRID(nnp_blocks((int64_t)n * (C / (32 * CPL)), tune.emb_block / 32)), tune.emb_block, 0, st, d))); }
    { NNP_PROF("k_embed_ln", st); nnp_launch((k_embed_ln<C>), NNP_GRID(warp_blocks), 256, 0, st, d); }
    {
        GemmBatch b{};
        b.g[0] = plain_gemm(d.ln0, m.es0_w, m.es0_b, d.e0, n, 2 * C, C);
        b.g[0].out2 = d.se0;
        { NNP_PROF("gemm_dense", st); RUN((gemm_launch<PRO_NONE, EPI_STORE_SILU>(b, 1, st))); }
        b.g[0] = plain_gemm(d.se0, m.es1_w, m.es1_b, d.e1, n, 3 * C, 2 * C);
        { NNP_PROF("gemm_dense", st); RUN((gemm_launch<PRO_NONE, EPI_STORE>(b, 1, st))); }
        if (L == 0) {
            GemmBatch mx = mix_gemm(d.X0, m.et_w, d.Xa, n, C, d.Xm, d.e1, 3 * C);
            { NNP_PROF("gemm_mix", st); RUN((gemm_launch<PRO_NONE, EPI_GATE>(mx, 3, st))); }
        } else {   // the gate is applied by the first layer's normalisation
            GemmBatch mx = mix_gemm(d.X0, m.et_w, d.Xm, n, C);
            { NNP_PROF("gemm_mix", st); RUN((gemm_launch<PRO_NONE, EPI_STORE>(mx, 3, st))); }
        }
    }
    float *X = d.Xa, *Xother = d.Xb;

    // ---- interaction layers
    for (int l = 0; l < L; ++l) {
        if (l == 0) { NNP_PROF("k_normalize", st); nnp_launch((k_normalize), NNP_GRID(ew_blocks), 256, 0, st, d.Xm, d.e1, d.Xh[l], d.nx[l], n, C); }
        GemmBatch my = mix_gemm(d.Xh[l], m.layer_t_w[l], d.Yc[l], n, C);
        { NNP_PROF("gemm_mix", st); RUN((gemm_launch<PRO_NONE, EPI_STORE>(my, 3, st))); }
        { NNP_PROF("k_edge_message", st); EDGE_DISPATCH(C, tune.fwd, (nnp_launch((k_edge_message_split<C, CPL>), NNP_GRID(nnp_blocks((int64_t)n * 2 * (C / (32 * CPL)), tune.fwd_block / 32)), tune.fwd_block, 0, st, d, l))); }
        GemmBatch md = mix_gemm(d.Qc, m.layer_t_w[l] + 3, d.Dc[l], n, C);
        { NNP_PROF("gemm_mix", st); RUN((gemm_launch<PRO_NONE, EPI_STORE>(md, 3, st))); }
        { NNP_PROF("k_residual", st); nnp_launch((k_residual), NNP_GRID(ew_blocks), 256, 0, st, d.Xh[l], d.Dc[l], Xother, l + 1 < L ? d.Xh[l + 1] : nullptr, l + 1 < L ? d.nx[l + 1] : nullptr, n, C); }
        std::swap(X, Xother);
    }

    // ---- readout
    { NNP_PROF("k_readout_feats", st); nnp_launch((k_readout_feats<C>), NNP_GRID(warp_blocks), 256, 0, st, d, X); }
    {
        GemmBatch b{};
        b.g[0] = plain_gemm(d.lnr, m.lin_w, m.lin_b, d.r0, n, C, 3 * C);
        b.g[0].out2 = d.sr0;
        { NNP_PROF("gemm_dense", st); RUN((gemm_launch<PRO_NONE, EPI_STORE_SILU>(b, 1, st))); }
        b.g[0] = plain_gemm(d.sr0, m.h1_w, m.h1_b, d.r1, n, H, C);
        { NNP_PROF("gemm_dense", st); RUN((gemm_launch<PRO_NONE, EPI_STORE>(b, 1, st))); }
    }
    { NNP_PROF("k_head", st); nnp_launch((k_head), NNP_GRID(warp_blocks), 256, 0, st, d, H); }
    { NNP_PROF("k_energy_sum", st); nnp_launch((k_energy_sum), NNP_GRID(d.n_samples), (n / d.n_samples >= 2048 ? 1024 : 256), 0, st, d); }
    NNP_CHECK_LAUNCH("tensornet forward");
    if (!d.forces) return NNP_OK;

    // ================================================================= reverse sweep
    {
        GemmBatch b{};
        // g_r0 = (g_r1 @ h1_w) * silu'(r0)
        b.g[0] = plain_gemm(d.g_r1, m.h1_wT, nullptr, d.g_r0, n, C, H, d.r0, C);
        { NNP_PROF("gemm_dense", st); RUN((gemm_launch<PRO_NONE, EPI_MUL_SILU_GRAD>(b, 1, st))); }
        b.g[0] = plain_gemm(d.g_r0, m.lin_wT, nullptr, d.g_lnr, n, 3 * C, C);
        { NNP_PROF("gemm_dense", st); RUN((gemm_launch<PRO_NONE, EPI_STORE>(b, 1, st))); }
    }
    // Three gradient buffers: GX = dL/dX of the layer above (kept until the normalisation's reverse,
    // which overwrites it in place), GB = G_D -> G_M -> next G_D (or G_Xm), GC = G_Q -> mixed-back G_Y.
    float *GX = d.G1, *GB = d.G2, *GC = d.G3;
    // GB = G_D of the last layer comes out of the readout's reverse (fused k_residual_bwd)
    { NNP_PROF("k_readout_bwd", st); nnp_launch((k_readout_bwd<C>), NNP_GRID(warp_blocks), 256, 0, st, d, X, GX, L > 0 ? d.Dc[L - 1] : nullptr, GB); }

    for (int l = L - 1; l >= 0; --l) {
        GemmBatch mq = mix_gemm(GB, m.layer_t_wT[l] + 3, GC, n, C);     // GC = G_Q
        { NNP_PROF("gemm_mix", st); RUN((gemm_launch<PRO_NONE, EPI_STORE>(mq, 3, st))); }
        { NNP_PROF("k_node_product_bwd", st); nnp_launch((k_node_product_bwd), NNP_GRID(ew_blocks), 256, 0, st, d.Mc[l], d.Yc[l], GC, GB, d.Qc, n, C); }
        // now GB = G_M, Qc = G_Y (local part)
        if (tune.bwd_split == 2) { NNP_PROF("k_edge_message_bwd", st); EDGE_DISPATCH(C, tune.bwd, (nnp_launch((k_edge_message_bwd_ring<C, CPL>), NNP_GRID(n), 64 * (C / (32 * CPL)), 0, st, d, l, GB, d.Qc, d.g_d + (size_t)(1 + l) * d.gd_slots * d.capacity))); }
        else if (tune.bwd_split) { NNP_PROF("k_edge_message_bwd", st); EDGE_DISPATCH(C, tune.bwd, (nnp_launch((k_edge_message_bwd_split<C, CPL>), NNP_GRID(nnp_blocks((int64_t)n * 2 * (C / (32 * CPL)), tune.bwd_block / 32)), tune.bwd_block, 0, st, d, l, GB, d.Qc, d.g_d + (size_t)(1 + l) * d.gd_slots * d.capacity))); }
        else { NNP_PROF("k_edge_message_bwd", st); EDGE_DISPATCH(C, tune.bwd, (nnp_launch((k_edge_message_bwd<C, CPL>), NNP_GRID(nnp_blocks((int64_t)n * (C / (32 * CPL)), tune.bwd_block / 32)), tune.bwd_block, 0, st, d, l, GB, d.Qc, d.g_d + (size_t)(1 + l) * d.gd_slots * d.capacity))); }
        // G_Xh = GX + mix^T(G_Y): the sum is formed by the normalisation's reverse, which also writes
        // what the next stage reads - G_D of layer l - 1, or the embedding gate's reverse at layer 0
        GemmBatch mh = mix_gemm(d.Qc, m.layer_t_wT[l], GC, n, C);
        { NNP_PROF("gemm_mix", st); RUN((gemm_launch<PRO_NONE, EPI_STORE>(mh, 3, st))); }
        if (l > 0) { NNP_PROF("k_normalize_bwd", st); nnp_launch((k_normalize_bwd), NNP_GRID(ew_blocks), 256, 0, st, GX, GC, d.Xh[l], d.nx[l], GX, d.Dc[l - 1], GB, nullptr, nullptr, nullptr, nullptr, n, C); }
        else { NNP_PROF("k_normalize_bwd", st); nnp_launch((k_normalize_bwd), NNP_GRID(ew_blocks), 256, 0, st, GX, GC, d.Xh[l], d.nx[l], nullptr, nullptr, nullptr, d.Xm, d.e1, GB, d.g_e1, n, C); }
    }
    // no interaction layer: X = Xm * gate went straight into the readout
    if (L == 0) { NNP_PROF("k_embed_gate_bwd", st); nnp_launch((k_embed_gate_bwd), NNP_GRID(ew_blocks), 256, 0, st, GX, d.Xm, d.e1, GB, d.g_e1, n, C); }

    // ---- embedding reverse: GB = G_Xm
    {
        GemmBatch b{};
        b.g[0] = plain_gemm(d.g_e1, m.es1_wT, nullptr, d.g_e0, n, 2 * C, 3 * C, d.e0, 2 * C);
        { NNP_PROF("gemm_dense", st); RUN((gemm_launch<PRO_NONE, EPI_MUL_SILU_GRAD>(b, 1, st))); }
        b.g[0] = plain_gemm(d.g_e0, m.es0_wT, nullptr, d.g_ln0, n, C, 2 * C);
        { NNP_PROF("gemm_dense", st); RUN((gemm_launch<PRO_NONE, EPI_STORE>(b, 1, st))); }
        GemmBatch mx = mix_gemm(GB, m.et_wT, GC, n, C);                                 // GC = G_X0 part
        { NNP_PROF("gemm_mix", st); RUN((gemm_launch<PRO_NONE, EPI_STORE>(mx, 3, st))); }
    }
    { NNP_PROF("k_embed_norm_bwd", st); nnp_launch((k_embed_norm_bwd<C>), NNP_GRID(warp_blocks), 256, 0, st, d, GC); }
    if (d.m.embed_projection) {
        // Hs = G_X0 against the sender-species weights, Hr against the receiver-species weights
        // (GB and GX are free by now); then one lane per edge
        nnp_gemm_weight ws[3], wr[3];
        for (int k = 0; k < 3; ++k) {
            ws[k].w = d.Wproj + (size_t)(k * 2 + 0) * EMB_SLOTS * EMB_K * C;
            wr[k].w = d.Wproj + (size_t)(k * 2 + 1) * EMB_SLOTS * EMB_K * C;
        }
        GemmBatch ms = mix_gemm(GC, ws, GB, n, C), mr = mix_gemm(GC, wr, GX, n, C);
        for (int k = 0; k < 3; ++k) {
            ms.g[k].N = mr.g[k].N = EMB_SLOTS * EMB_K;
            ms.g[k].ldo = mr.g[k].ldo = EMB_SLOTS * EMB_K;
        }
        { NNP_PROF("gemm_embed_proj", st); RUN((gemm_launch<PRO_NONE, EPI_STORE>(ms, 3, st))); }
        { NNP_PROF("gemm_embed_proj", st); RUN((gemm_launch<PRO_NONE, EPI_STORE>(mr, 3, st))); }
        { NNP_PROF("k_embed_edge_bwd_proj", st); nnp_launch((k_embed_edge_bwd_proj), NNP_GRID(nnp_blocks(n, EMB_PROJ_WARPS)), EMB_PROJ_WARPS * 32, 0, st, d, GB, GX); }
    }
    // (a knot-cached variant of this fallback was measured slower: 1.62 vs 1.34 ms at config D, 22.9 vs 20.9 us at A)
    { NNP_PROF("k_embed_edge_bwd", st); EDGE_DISPATCH(C, tune.embbwd, (nnp_launch((k_embed_edge_bwd<C, CPL>), NNP_GRID(nnp_blocks((int64_t)n * (C / (32 * CPL)), tune.emb_block / 32)), tune.emb_block, 0, st, d, GC))); }
    { NNP_PROF("k_forces", st); nnp_launch((k_forces), NNP_GRID(warp_blocks), 256, 0, st, d); }
    NNP_CHECK_LAUNCH("tensornet reverse");
#undef RUN
    return NNP_OK;
}

}  // namespace

extern "C" int nnp_tn_workspace_bytes(const nnp_tn_model *m, int32_t n_atoms, int32_t capacity,
                                      int32_t n_samples, size_t *bytes)
{
    int rc = validate_model(m);
    if (rc) return rc;
    NNP_CHECK_ARG(n_atoms >= 1 && capacity >= 1 && n_samples >= 1 && bytes, "bad sizes");
    TnDev d{};
    d.m = *m;
    d.n = n_atoms;
    d.capacity = capacity;
    d.n_samples = n_samples;
    *bytes = carve(d, nullptr);
    return NNP_OK;
}

extern "C" int nnp_tn_energy_forces(const nnp_tn_model *m, int32_t n_atoms, int32_t n_samples,
                                    int32_t capacity, const int32_t *species, const int32_t *batch,
                                    const int32_t *order, const int32_t *row_ptr,
                                    const int32_t *pairs, const float *deltas, const float *dists,
                                    const int32_t *nl_counts, float *energy, float *forces,
                                    float *per_atom, void *workspace, size_t workspace_bytes,
                                    nnp_stream_t stream)
{
    int rc = validate_model(m);
    if (rc) return rc;
    NNP_CHECK_ARG(n_atoms >= 1 && capacity >= 1 && n_samples >= 1, "bad sizes");
    NNP_CHECK_ARG(species && batch && row_ptr && pairs && deltas && dists && energy && workspace,
                  "NULL buffer passed to nnp_tn_energy_forces");
    TnDev d{};
    d.m = *m;
    d.n = n_atoms;
    d.capacity = capacity;
    d.n_samples = n_samples;
    size_t need = carve(d, workspace);
    if (need > workspace_bytes) {
        nnp_set_error("workspace too small: need %zu bytes, got %zu", need, workspace_bytes);
        return NNP_ERR_WORKSPACE;
    }
    d.species = species;
    d.batch = batch;
    d.order = order;
    d.row_ptr = row_ptr;
    d.pairs = pairs;
    d.deltas = deltas;
    d.dists = dists;
    d.nl_counts = nl_counts;
    d.energy = energy;
    d.forces = forces;
    d.per_atom = per_atom;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    t_nnp_gemm_mode = m->gemm_mode == 0 ? g_gemm_default.load(std::memory_order_relaxed)
                                        : (m->gemm_mode == 8 ? 0 : m->gemm_mode);
    switch (m->channels) {
    case 32: return run_step<32>(d, st);
    case 64: return run_step<64>(d, st);
    default: return run_step<128>(d, st);
    }
}

extern "C" int nnp_set_gemm_mode(int use_mma)
{
    g_gemm_default.store((use_mma == 5 || use_mma == 3 || use_mma == 1) ? use_mma : (use_mma <= 0 ? 0 : 5));
    return NNP_OK;
}

extern "C" int nnp_test_gemm_nt(const float *A, const nnp_gemm_weight *W, const float *bias,
                                float *out, int32_t M, int32_t N, int32_t K, nnp_stream_t stream)
{
    NNP_CHECK_ARG(A && W && W->w && out && M >= 1 && N >= 1 && K >= 4,
                  "bad arguments to nnp_test_gemm_nt");
    GemmBatch b{};
    b.g[0] = plain_gemm(A, *W, bias, out, M, N, K);
    t_nnp_gemm_mode = g_gemm_default.load(std::memory_order_relaxed);
    return gemm_launch<PRO_NONE, EPI_STORE>(b, 1, static_cast<cudaStream_t>(stream));
}
