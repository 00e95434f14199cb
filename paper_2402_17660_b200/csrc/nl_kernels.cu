// Cutoff neighbor search for sm_100a: cell binning, deterministic counting sort of atoms by
// cell, and a warp-per-atom scan of the 27 surrounding cells (or of the atom's own sample for
// the brute strategy) that emits a CSR structure sorted by (i, j).
//
// Replaces, with identical results, the reference's
//   neighbors.py:103-133   grid construction + cell sort
//   _neighbor_kernels.py:24-233   brute/cell x open/wrapped pair kernels
//   neighbors.py:204-225   overflow count, full-list mirror, self loops, lexsort
//
// Exactness: every accept/reject decision and every emitted delta/distance is computed in
// float64 with the reference's operation order (d = r_i - r_j for i < j, reduce c then b
// then a with rint(component/diagonal), d2 = (dx*dx + dy*dy) + dz*dz, window on squared
// distances) using __dmul_rn/__dadd_rn/__dsub_rn so that no FMA is contracted.  Mirrored rows
// (j, i) are the exact negation, as in neighbors.py:209-212.
//
// Two passes over the candidates (count -> exclusive scan -> fill) give each row its final
// offset without atomics, so the output order is deterministic and equals np.lexsort((j, i)).
#include <algorithm>
#include <cmath>

#include "nnp_common.cuh"

namespace {

constexpr int NL_THREADS = 256;
constexpr int NL_WARPS = NL_THREADS / 32;
constexpr int NL_MAXROW = 256;  // row entries kept in shared memory; longer rows use scratch

struct GridDev {
    int dims[3];
    int ncell;
    double low[3];
    double inv_edge[3];
    // the row scan's single-precision screen: Cartesian step between adjacent cells along each grid
    // axis, and the squared-distance window widened by the screen's error bound
    float cv[3][3];
    float hi2w, lo2w;
    // cell culling: fractional position of a point inside its cell from its local Cartesian coordinates
    // (back substitution through the lower-triangular cell vectors), the cell's perpendicular widths,
    // and whether the three widths are orthogonal (then the gaps to a neighbour cell add in quadrature)
    float wid[3];
    float icv[3];      // 1 / cv[k][k]
    float cull2;       // squared reach beyond which a whole neighbour cell cannot hold a pair (widened)
    int ortho;
};

struct Metric {
    int wrapped;
    double b00, b10, b11, b20, b21, b22;
    double i00, i11, i22;
    double lo2, hi2;
};

// float copy of the metric for the prefilter; hi2p / lo2m are the window widened by the
// prefilter's error bound (relative eps of the squared distance)
struct MetricF {
    float b00, b10, b11, b20, b21, b22, i00, i11, i22, hi2p, lo2m;
};

struct NlArgs {
    int n, n_samples, capacity, strategy, flags, periodic, max_cells;
    int stage_w;      // accepted candidates kept per row between the count and the fill pass
    MetricF mf;
    double cutoff;
    double inv_box[9];
    int host_dims[3];
    Metric metric;
    const double *pos;
    const int *batch;
    // workspace
    int *cell_id, *cell_start, *cell_cursor, *tmp_order, *sidx, *rank_of, *sbatch, *row_count;
    int *sample_ptr, *scratch_col, *scratch_t, *stage_t;
    double *spos;
    float4 *slpos;   // cell strategy: (position relative to the atom's own cell corner, original index)
    int4 *scell;     // cell strategy: grid coordinates of the sorted atom's cell (and the flat index): the row
                     // scan needs them per atom and a division by a runtime grid size costs ~25 instructions
    double *bounds_partial;
    GridDev *grid;
    // outputs
    int *pairs, *row_ptr, *order, *counts;
    void *deltas, *dists;
};

__device__ __forceinline__ double rint_div(double x, double diag, double inv_diag)
{
    double q = x * inv_diag;
    double r = rint(q);
    // the reciprocal product can only disagree with the true quotient next to a tie
    if (fabs(fabs(q - r) - 0.5) < 1e-6) r = rint(x / diag);
    return r;
}

// Displacement r_lo - r_hi of the pair ordered by ORIGINAL index (as the reference computes
// it), reduced to the minimum image; returns the squared norm.
__device__ __forceinline__ double pair_delta(const Metric &m, double ax, double ay, double az,
                                             double bx, double by, double bz, double &dx,
                                             double &dy, double &dz)
{
    dx = __dsub_rn(ax, bx);
    dy = __dsub_rn(ay, by);
    dz = __dsub_rn(az, bz);
    if (m.wrapped) {
        double s = rint_div(dz, m.b22, m.i22);
        dx = __dsub_rn(dx, __dmul_rn(s, m.b20));
        dy = __dsub_rn(dy, __dmul_rn(s, m.b21));
        dz = __dsub_rn(dz, __dmul_rn(s, m.b22));
        s = rint_div(dy, m.b11, m.i11);
        dx = __dsub_rn(dx, __dmul_rn(s, m.b10));
        dy = __dsub_rn(dy, __dmul_rn(s, m.b11));
        dx = __dsub_rn(dx, __dmul_rn(m.b00, rint_div(dx, m.b00, m.i00)));
    }
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// sample_ptr[b] = first atom of sample b (batch is non-decreasing, system.py:231-235)
__global__ void k_sample_ptr(const int *__restrict__ batch, int n, int n_samples,
                             int *__restrict__ sample_ptr, int *__restrict__ counts)
{
    NNP_PDL_SYNC();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < 4) counts[b] = 0;
    if (b > n_samples) return;
    int lo = 0, hi = n;
    if (n_samples == 1) lo = hi = (b == 0 ? 0 : n);      // one sample: no search (15 dependent loads)
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (batch[mid] < b) lo = mid + 1; else hi = mid;
    }
    sample_ptr[b] = lo;
}

// ---- open-boundary grid: bounding box reduction (neighbors.py:116-124)
__global__ void k_bounds_partial(const double *__restrict__ pos, int n, double *__restrict__ partial)
{
    NNP_PDL_SYNC();
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double v = pos[3 * (size_t)i + k];
            lo[k] = fmin(lo[k], v);
            hi[k] = fmax(hi[k], v);
        }
    }
    __shared__ double s[NL_WARPS][6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        for (int o = 16; o > 0; o >>= 1) {
            lo[k] = fmin(lo[k], __shfl_xor_sync(NNP_FULL_MASK, lo[k], o));
            hi[k] = fmax(hi[k], __shfl_xor_sync(NNP_FULL_MASK, hi[k], o));
        }
    }
    if ((threadIdx.x & 31) == 0) {
        for (int k = 0; k < 3; ++k) {
            s[threadIdx.x >> 5][k] = lo[k];
            s[threadIdx.x >> 5][3 + k] = hi[k];
        }
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        double v = s[0][threadIdx.x];
        for (int w = 1; w < NL_WARPS; ++w)
            v = threadIdx.x < 3 ? fmin(v, s[w][threadIdx.x]) : fmax(v, s[w][threadIdx.x]);
        partial[blockIdx.x * 6 + threadIdx.x] = v;
    }
}

__global__ void k_grid_setup(NlArgs a, int n_partial)
{
    NNP_PDL_SYNC();
    if (threadIdx.x != 0) return;
    GridDev g;
    if (a.periodic) {
        for (int k = 0; k < 3; ++k) {
            g.dims[k] = a.host_dims[k];
            g.low[k] = 0.0;
            g.inv_edge[k] = 0.0;
        }
    } else {
        double lo[3], hi[3];
        for (int k = 0; k < 3; ++k) {
            lo[k] = a.bounds_partial[k];
            hi[k] = a.bounds_partial[3 + k];
        }
        for (int b = 1; b < n_partial; ++b)
            for (int k = 0; k < 3; ++k) {
                lo[k] = fmin(lo[k], a.bounds_partial[b * 6 + k]);
                hi[k] = fmax(hi[k], a.bounds_partial[b * 6 + 3 + k]);
            }
        double extent[3];
        for (int k = 0; k < 3; ++k) {
            g.low[k] = lo[k] - 0.5 * a.cutoff;
            extent[k] = hi[k] - g.low[k] + 0.5 * a.cutoff;
            double d = floor(extent[k] / a.cutoff);
            g.dims[k] = d < 1.0 ? 1 : (d > 1.0e6 ? 1000000 : (int)d);
        }
        // never more cells than the workspace holds: coarsen the longest axis (cells only grow,
        // so the 27-cell neighbourhood still covers the cutoff)
        while ((int64_t)g.dims[0] * g.dims[1] * g.dims[2] > (int64_t)a.max_cells) {
            int k = 0;
            if (g.dims[1] > g.dims[k]) k = 1;
            if (g.dims[2] > g.dims[k]) k = 2;
            g.dims[k] = (g.dims[k] + 1) / 2;
        }
        for (int k = 0; k < 3; ++k) g.inv_edge[k] = (double)g.dims[k] / extent[k];
    }
    g.ncell = g.dims[0] * g.dims[1] * g.dims[2];
    {
        const Metric &m = a.metric;
        double cv[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        if (a.periodic) {
            cv[0][0] = m.b00 / g.dims[0];
            cv[1][0] = m.b10 / g.dims[1]; cv[1][1] = m.b11 / g.dims[1];
            cv[2][0] = m.b20 / g.dims[2]; cv[2][1] = m.b21 / g.dims[2]; cv[2][2] = m.b22 / g.dims[2];
        } else {
            for (int k = 0; k < 3; ++k) cv[k][k] = 1.0 / g.inv_edge[k];
        }
        double ext = 0.0;
        for (int k = 0; k < 3; ++k) {
            ext += sqrt(cv[k][0] * cv[k][0] + cv[k][1] * cv[k][1] + cv[k][2] * cv[k][2]);
            for (int c = 0; c < 3; ++c) g.cv[k][c] = (float)cv[k][c];
        }
        // local coordinates, shift and their differences are each good to 2^-24 of the cell's
        // extent: 8 roundings per component, x sqrt(3), x 5 margin
        const double slack = 4.0e-6 * ext;
        const double r_hi = sqrt(m.hi2) * 1.000001 + slack, r_lo = sqrt(m.lo2) * 0.999999 - slack;
        g.hi2w = (float)(r_hi * r_hi * 1.000002);
        g.lo2w = r_lo > 0.0 ? (float)(r_lo * r_lo * 0.999998) : -1.0f;
        // perpendicular widths of a cell: 1 / |gradient of the fractional coordinate|
        const double c00 = cv[0][0], c10 = cv[1][0], c11 = cv[1][1], c20 = cv[2][0], c21 = cv[2][1], c22 = cv[2][2];
        const double g0[3] = {1.0 / c00, -c10 / (c00 * c11), (c10 * c21 - c20 * c11) / (c00 * c11 * c22)};
        const double g1[3] = {0.0, 1.0 / c11, -c21 / (c11 * c22)};
        g.wid[0] = (float)(1.0 / sqrt(g0[0] * g0[0] + g0[1] * g0[1] + g0[2] * g0[2]));
        g.wid[1] = (float)(1.0 / sqrt(g1[1] * g1[1] + g1[2] * g1[2]));
        g.wid[2] = (float)c22;
        g.icv[0] = (float)(1.0 / c00);
        g.icv[1] = (float)(1.0 / c11);
        g.icv[2] = (float)(1.0 / c22);
        g.ortho = (c10 == 0.0 && c20 == 0.0 && c21 == 0.0) ? 1 : 0;
        // a cell is skipped when even its nearest plane is farther than the cutoff plus 0.1 % of a
        // cell (three orders above the float32 error of the local coordinates)
        const double reach = r_hi + 1.0e-3 * ext;
        g.cull2 = (float)(reach * reach);
    }
    *a.grid = g;
    a.counts[2] = g.ncell;
}

__global__ void k_cell_assign(NlArgs a)
{
    NNP_PDL_SYNC();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    const GridDev g = *a.grid;
    double x = a.pos[3 * (size_t)i], y = a.pos[3 * (size_t)i + 1], z = a.pos[3 * (size_t)i + 2];
    int c[3];
    if (a.periodic) {
        // fractional coordinates, wrapped into [0,1)  (neighbors.py:110-112)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double f = x * a.inv_box[k] + y * a.inv_box[3 + k] + z * a.inv_box[6 + k];
            f -= floor(f);
            int v = (int)floor(f * g.dims[k]);
            c[k] = v < 0 ? 0 : (v >= g.dims[k] ? g.dims[k] - 1 : v);
        }
    } else {
        double p[3] = {x, y, z};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            int v = (int)floor((p[k] - g.low[k]) * g.inv_edge[k]);
            c[k] = v < 0 ? 0 : (v >= g.dims[k] ? g.dims[k] - 1 : v);
        }
    }
    int flat = (c[0] * g.dims[1] + c[1]) * g.dims[2] + c[2];
    a.cell_id[i] = flat;
    atomicAdd(&a.cell_start[flat], 1);  // counts; turned into starts by the scan that follows
}

__global__ void k_cell_scatter(NlArgs a)
{
    NNP_PDL_SYNC();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    int c = a.cell_id[i];
    int slot = a.cell_start[c] + atomicAdd(&a.cell_cursor[c], 1);
    a.tmp_order[slot] = i;
}

// Stable order inside each cell (ascending original index), so the sort equals
// np.argsort(flat, kind="stable") (neighbors.py:129) whatever order the atomics ran in.
__global__ void k_cell_rank(NlArgs a)
{
    NNP_PDL_SYNC();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    int c = a.cell_id[i];
    int p0 = a.cell_start[c], p1 = a.cell_start[c + 1];
    int rank = 0;
    for (int t = p0; t < p1; ++t) rank += (a.tmp_order[t] < i);
    int s = p0 + rank;
    a.sidx[s] = i;
    a.rank_of[i] = s;
    if (a.order) a.order[s] = (a.flags & NNP_NL_RENUMBER) ? i : s;
    a.sbatch[s] = a.batch[i];
    a.spos[3 * (size_t)s] = a.pos[3 * (size_t)i];
    a.spos[3 * (size_t)s + 1] = a.pos[3 * (size_t)i + 1];
    a.spos[3 * (size_t)s + 2] = a.pos[3 * (size_t)i + 2];
    // Single-precision position relative to the corner of the atom's own cell (computed in float64,
    // so its error is 2^-24 of a cell edge whatever the size of the box); the row scan's prefilter
    // rebuilds the displacement to a candidate in an adjacent cell as
    //   (local_a - local_b) - (cell offset) . (cell vectors).
    const GridDev g = *a.grid;
    const double x = a.pos[3 * (size_t)i], y = a.pos[3 * (size_t)i + 1], z = a.pos[3 * (size_t)i + 2];
    const int cc[3] = {c / (g.dims[1] * g.dims[2]), (c / g.dims[2]) % g.dims[1], c % g.dims[2]};
    a.scell[s] = make_int4(cc[0], cc[1], cc[2], c);
    double lx, ly, lz;
    if (a.periodic) {
        double w[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double f = x * a.inv_box[k] + y * a.inv_box[3 + k] + z * a.inv_box[6 + k];
            f -= floor(f);
            w[k] = (f * g.dims[k] - cc[k]) / g.dims[k];     // fraction of the box edge past the cell corner
        }
        const Metric &m = a.metric;
        lx = w[0] * m.b00 + w[1] * m.b10 + w[2] * m.b20;
        ly = w[1] * m.b11 + w[2] * m.b21;
        lz = w[2] * m.b22;
    } else {
        lx = x - g.low[0] - cc[0] / g.inv_edge[0];
        ly = y - g.low[1] - cc[1] / g.inv_edge[1];
        lz = z - g.low[2] - cc[2] / g.inv_edge[2];
    }
    a.slpos[s] = make_float4((float)lx, (float)ly, (float)lz, __int_as_float(i));
}

__global__ void k_identity_order(NlArgs a)
{
    NNP_PDL_SYNC();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    a.sidx[i] = i;
    a.rank_of[i] = i;
    if (a.order) a.order[i] = i;
    a.sbatch[i] = a.batch[i];
    a.spos[3 * (size_t)i] = a.pos[3 * (size_t)i];
    a.spos[3 * (size_t)i + 1] = a.pos[3 * (size_t)i + 1];
    a.spos[3 * (size_t)i + 2] = a.pos[3 * (size_t)i + 2];
}

// Candidate runs [p0, p1) in sorted-atom space for the atom at sorted position s.
template <typename F>
__device__ __forceinline__ void visit_runs(const NlArgs &a, const GridDev &g, int cell, int bi, F &&f)
{
    if (a.strategy == NNP_STRATEGY_BRUTE) {
        // same-sample atoms are contiguous (system.py:231-235); foreign samples can never pair
        f(a.sample_ptr[bi], a.sample_ptr[bi + 1]);
        return;
    }
    const int m0 = g.dims[0], m1 = g.dims[1], m2 = g.dims[2];
    const int c2 = cell % m2;
    const int c1 = (cell / m2) % m1;
    const int c0 = cell / (m1 * m2);
    for (int o0 = -1; o0 <= 1; ++o0) {
        int n0 = c0 + o0;
        if (a.periodic) {
            n0 = n0 < 0 ? n0 + m0 : (n0 >= m0 ? n0 - m0 : n0);
        } else if (n0 < 0 || n0 >= m0) {
            continue;
        }
        for (int o1 = -1; o1 <= 1; ++o1) {
            int n1 = c1 + o1;
            if (a.periodic) {
                n1 = n1 < 0 ? n1 + m1 : (n1 >= m1 ? n1 - m1 : n1);
            } else if (n1 < 0 || n1 >= m1) {
                continue;
            }
            const int base = (n0 * m1 + n1) * m2;
            int lo = c2 - 1, hi = c2 + 1;
            if (a.periodic) {
                // three cells along the fastest axis are contiguous in the sorted order except
                // where they wrap (the periodic grid has >= 3 cells per axis)
                if (lo < 0) {
                    f(a.cell_start[base + m2 - 1], a.cell_start[base + m2]);
                    lo = 0;
                }
                if (hi >= m2) {
                    f(a.cell_start[base], a.cell_start[base + 1]);
                    hi = m2 - 1;
                }
            } else {
                lo = lo < 0 ? 0 : lo;
                hi = hi >= m2 ? m2 - 1 : hi;
            }
            f(a.cell_start[base + lo], a.cell_start[base + hi + 1]);
        }
    }
}

// Cheap single-precision screen of a candidate: the coordinate differences are taken in float64
// (exact to 1 ulp whatever the magnitude of the coordinates) and everything after that runs in
// float32 against a window widened by the error bound.  Only survivors get the exact float64
// evaluation, which alone decides membership and produces the output values.
__device__ __forceinline__ bool prefilter(const NlArgs &a, double ax, double ay, double az, double bx,
                                          double by, double bz)
{
    float fx = (float)(ax - bx), fy = (float)(ay - by), fz = (float)(az - bz);
    const MetricF &m = a.mf;
    if (a.periodic) {
        float sft = rintf(fz * m.i22);
        fx -= sft * m.b20;
        fy -= sft * m.b21;
        fz -= sft * m.b22;
        sft = rintf(fy * m.i11);
        fx -= sft * m.b10;
        fy -= sft * m.b11;
        fx -= m.b00 * rintf(fx * m.i00);
    }
    const float d2 = fx * fx + fy * fy + fz * fz;
    return d2 <= m.hi2p && d2 >= m.lo2m;
}

template <bool FILL, typename OutT>
__global__ void __launch_bounds__(NL_THREADS, FILL ? 6 : 0) k_rows(NlArgs a)
{
    NNP_PDL_SYNC();
    __shared__ int s_col[FILL ? NL_WARPS : 1][FILL ? NL_MAXROW : 1];
    __shared__ int s_t[FILL ? NL_WARPS : 1][FILL ? NL_MAXROW : 1];
    __shared__ int s_queue[NL_WARPS][64];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int s = blockIdx.x * NL_WARPS + wib;
    if (s >= a.n) return;
    if (FILL) {
        const int total = a.row_ptr[a.n];
        if (s == 0 && lane == 0) a.counts[0] = total;
        if (total > a.capacity) return;          // overflow: the host raises CapacityError
    } else if (s == 0 && lane == 0) {
        a.row_count[a.n] = 0;                     // so that the scan's last output is the total
    }

    const bool full = a.flags & NNP_NL_FULL_LIST;
    const bool renumber = a.flags & NNP_NL_RENUMBER;
    const int io = a.sidx[s];
    const int bi = a.sbatch[s];
    const int row = renumber ? s : io;
    const double ax = a.spos[3 * (size_t)s], ay = a.spos[3 * (size_t)s + 1],
                 az = a.spos[3 * (size_t)s + 2];
    const Metric m = a.metric;
    int *queue = s_queue[wib];
    int *stage = a.stage_t + (size_t)s * a.stage_w;

    int *list_col = nullptr, *list_t = nullptr;
    int row_start = 0;
    bool from_stage = false;
    int cnt = 0;
    if (FILL) {
        row_start = a.row_ptr[row];
        const int expect = a.row_ptr[row + 1] - row_start;
        if (expect <= NL_MAXROW) {
            list_col = s_col[wib];
            list_t = s_t[wib];
        } else {
            list_col = a.scratch_col + row_start;
            list_t = a.scratch_t + row_start;
        }
        if (expect <= a.stage_w) {
            // the count pass kept this row's accepted candidates: no second scan
            from_stage = true;
            for (int e = lane; e < expect; e += 32) {
                const int t = stage[e];
                list_t[e] = t;
                list_col[e] = renumber ? t : a.sidx[t];
            }
            cnt = expect;
        }
    }

    if (!from_stage) {
        const unsigned lt_mask = (1u << lane) - 1u;
        int qn = 0;
        // exact float64 test of up to 32 queued candidates (one per lane)
        auto exact_step = [&](int t, bool valid) {
            bool ok = false;
            int jo = 0;
            if (valid) {
                jo = a.sidx[t];
                const double bx = a.spos[3 * (size_t)t], by = a.spos[3 * (size_t)t + 1],
                             bz = a.spos[3 * (size_t)t + 2];
                double dx, dy, dz, d2;
                if (io < jo)
                    d2 = pair_delta(m, ax, ay, az, bx, by, bz, dx, dy, dz);
                else
                    d2 = pair_delta(m, bx, by, bz, ax, ay, az, dx, dy, dz);
                ok = d2 > m.lo2 && d2 <= m.hi2;
            }
            const unsigned hit = __ballot_sync(NNP_FULL_MASK, ok);
            if (ok) {
                const int p = cnt + __popc(hit & lt_mask);
                if (FILL) {
                    list_col[p] = renumber ? t : jo;
                    list_t[p] = t;
                } else if (p < a.stage_w) {
                    stage[p] = t;
                }
            }
            cnt += __popc(hit);
        };
        auto process = [&](int p0, int p1) {
            for (int base = p0; base < p1; base += 32) {
                const int t = base + lane;
                bool pass = false;
                if (t < p1) {
                    const int jo = a.sidx[t];
                    if (a.sbatch[t] == bi && jo != io && (full || jo > io))
                        pass = prefilter(a, ax, ay, az, a.spos[3 * (size_t)t],
                                         a.spos[3 * (size_t)t + 1], a.spos[3 * (size_t)t + 2]);
                }
                const unsigned mk = __ballot_sync(NNP_FULL_MASK, pass);
                if (pass) queue[qn + __popc(mk & lt_mask)] = t;
                qn += __popc(mk);
                __syncwarp();
                if (qn >= 32) {
                    const int tq = queue[qn - 32 + lane];
                    qn -= 32;
                    exact_step(tq, true);
                    __syncwarp();
                }
            }
        };
        if (a.strategy == NNP_STRATEGY_CELL) {
            // The 27 surrounding cells as ONE candidate stream: lane r < 27 looks up cell r's run in
            // the sorted order and the displacement of its corner from the own cell's (the adjacent
            // periodic image where the neighbourhood wraps, so no rounding to the minimum image is
            // needed); every iteration then screens 32 consecutive candidates of the concatenated
            // runs, whatever cell boundaries fall between them.
            const GridDev g = *a.grid;
            const int4 cc = a.scell[s];
            const int m0 = g.dims[0], m1 = g.dims[1], m2 = g.dims[2];
            int r_start = 0, r_len = 0;
            float sh_x = 0.0f, sh_y = 0.0f, sh_z = 0.0f;
            const float4 la = a.slpos[s];
            if (lane < 27) {
                const int o0 = lane / 9 - 1, o1 = (lane / 3) % 3 - 1, o2 = lane % 3 - 1;
                int n0 = cc.x + o0, n1 = cc.y + o1, n2 = cc.z + o2;
                bool inside = true;
                if (a.periodic) {
                    n0 = n0 < 0 ? n0 + m0 : (n0 >= m0 ? n0 - m0 : n0);
                    n1 = n1 < 0 ? n1 + m1 : (n1 >= m1 ? n1 - m1 : n1);
                    n2 = n2 < 0 ? n2 + m2 : (n2 >= m2 ? n2 - m2 : n2);
                } else {
                    inside = n0 >= 0 && n0 < m0 && n1 >= 0 && n1 < m1 && n2 >= 0 && n2 < m2;
                }
                if (inside) {
                    // Cull cells that lie wholly beyond the cutoff of THIS atom: the neighbour cell in
                    // direction o along axis k starts at a plane whose perpendicular distance is
                    // (1 - f_k) w_k (o = +1) or f_k w_k (o = -1), f = fractional position in the own cell.
                    const float f2 = la.z * g.icv[2];
                    const float f1 = (la.y - f2 * g.cv[2][1]) * g.icv[1];
                    const float f0 = (la.x - f1 * g.cv[1][0] - f2 * g.cv[2][0]) * g.icv[0];
                    const float gap0 = o0 == 0 ? 0.0f : fmaxf(o0 > 0 ? 1.0f - f0 : f0, 0.0f) * g.wid[0];
                    const float gap1 = o1 == 0 ? 0.0f : fmaxf(o1 > 0 ? 1.0f - f1 : f1, 0.0f) * g.wid[1];
                    const float gap2 = o2 == 0 ? 0.0f : fmaxf(o2 > 0 ? 1.0f - f2 : f2, 0.0f) * g.wid[2];
                    const float far2 = g.ortho ? gap0 * gap0 + gap1 * gap1 + gap2 * gap2
                                               : fmaxf(gap0, fmaxf(gap1, gap2)) * fmaxf(gap0, fmaxf(gap1, gap2));
                    if (far2 <= g.cull2) {
                        const int flat = (n0 * m1 + n1) * m2 + n2;
                        r_start = a.cell_start[flat];
                        r_len = a.cell_start[flat + 1] - r_start;
                    }
                }
                sh_x = o0 * g.cv[0][0] + o1 * g.cv[1][0] + o2 * g.cv[2][0];
                sh_y = o0 * g.cv[0][1] + o1 * g.cv[1][1] + o2 * g.cv[2][1];
                sh_z = o0 * g.cv[0][2] + o1 * g.cv[1][2] + o2 * g.cv[2][2];
            }
            int incl = r_len;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int up = __shfl_up_sync(NNP_FULL_MASK, incl, d);
                if (lane >= d) incl += up;
            }
            const int total = __shfl_sync(NNP_FULL_MASK, incl, 31);
            // Lane r keeps run r's start, exclusive prefix and corner shift in registers; a candidate's
            // run is found without memory: runs are contiguous stretches of the stream, so the 32
            // candidates of an iteration span the run that holds the first of them plus the few runs
            // that begin inside the iteration (two ballots, then one shuffle per such run).
            const int my_pref = lane < 27 ? incl - r_len : 0x7fffffff;   // sentinel past the last run
            const float hi2w = g.hi2w, lo2w = g.lo2w;     // window widened by the screen's error bound
            const bool one_sample = a.n_samples == 1;
            for (int base = 0; base < total; base += 32) {
                const int idx = base + lane;
                const unsigned le = __ballot_sync(NNP_FULL_MASK, my_pref <= base);
                unsigned inside_mask = __ballot_sync(NNP_FULL_MASK, my_pref > base && my_pref <= base + 31);
                int r = 31 - __clz(le);                                   // last run that starts at or before base
                while (inside_mask) {
                    const int b = __ffs(inside_mask) - 1;
                    inside_mask &= inside_mask - 1;
                    if (__shfl_sync(NNP_FULL_MASK, my_pref, b) <= idx) r = b;
                }
                const int rs = __shfl_sync(NNP_FULL_MASK, r_start, r), rp = __shfl_sync(NNP_FULL_MASK, my_pref, r);
                const float sx = __shfl_sync(NNP_FULL_MASK, sh_x, r), sy = __shfl_sync(NNP_FULL_MASK, sh_y, r),
                            sz = __shfl_sync(NNP_FULL_MASK, sh_z, r);
                bool pass = false;
                int t = 0;
                if (idx < total) {
                    t = rs + (idx - rp);
                    const float4 lb = a.slpos[t];
                    const int jo = __float_as_int(lb.w);
                    if ((one_sample || a.sbatch[t] == bi) && jo != io && (full || jo > io)) {
                        const float fx = (la.x - lb.x) - sx;
                        const float fy = (la.y - lb.y) - sy;
                        const float fz = (la.z - lb.z) - sz;
                        const float d2 = fx * fx + fy * fy + fz * fz;
                        pass = d2 <= hi2w && d2 >= lo2w;
                    }
                }
                const unsigned mk = __ballot_sync(NNP_FULL_MASK, pass);
                if (pass) queue[qn + __popc(mk & lt_mask)] = t;
                qn += __popc(mk);
                __syncwarp();
                if (qn >= 32) {
                    const int tq = queue[qn - 32 + lane];
                    qn -= 32;
                    exact_step(tq, true);
                    __syncwarp();
                }
            }
        } else {
            GridDev g{};
            visit_runs(a, g, 0, bi, process);
        }
        if (qn > 0) {
            const bool valid = lane < qn;
            exact_step(valid ? queue[lane] : 0, valid);
        }
        if (a.flags & NNP_NL_SELF_LOOPS) {
            if (lane == 0) {
                if (FILL) {
                    list_col[cnt] = row;
                    list_t[cnt] = s;
                } else if (cnt < a.stage_w) {
                    stage[cnt] = s;
                }
            }
            cnt += 1;
        }
    }

    if (!FILL) {
        if (lane == 0) {
            a.row_count[row] = cnt;
            atomicMax(&a.counts[1], cnt);
        }
        return;
    }

    __syncwarp();
    OutT *deltas = static_cast<OutT *>(a.deltas);
    OutT *dists = static_cast<OutT *>(a.dists);
    for (int e = lane; e < cnt; e += 32) {
        const int col = ((volatile int *)list_col)[e];
        const int t = ((volatile int *)list_t)[e];
        int rank = e;                                   // NNP_NL_UNSORTED: the order of discovery
        if (!(a.flags & NNP_NL_UNSORTED)) {
            rank = 0;
            for (int q = 0; q < cnt; ++q) rank += (((volatile int *)list_col)[q] < col);
        }
        const size_t idx = (size_t)row_start + rank;
        a.pairs[2 * idx] = row;
        a.pairs[2 * idx + 1] = col;
        double dx = 0.0, dy = 0.0, dz = 0.0, dist = 0.0;
        if (t != s) {
            const int jo = a.sidx[t];
            const double bx = a.spos[3 * (size_t)t], by = a.spos[3 * (size_t)t + 1],
                         bz = a.spos[3 * (size_t)t + 2];
            double d2;
            if (io < jo) {
                d2 = pair_delta(m, ax, ay, az, bx, by, bz, dx, dy, dz);
            } else {
                d2 = pair_delta(m, bx, by, bz, ax, ay, az, dx, dy, dz);
                dx = -dx;
                dy = -dy;
                dz = -dz;
            }
            dist = sqrt(d2);
        }
        deltas[3 * idx] = (OutT)dx;
        deltas[3 * idx + 1] = (OutT)dy;
        deltas[3 * idx + 2] = (OutT)dz;
        dists[idx] = (OutT)dist;
    }
}

template <typename OutT>
__global__ void k_pad_tail(NlArgs a)
{
    NNP_PDL_SYNC();
    // fixed grid, element-wise over the three tails (the row count is only known on the device, so a
    // grid sized for the whole capacity would launch mostly idle blocks)
    const int total = a.row_ptr[a.n];
    if (total > a.capacity) return;
    const int64_t rows = (int64_t)a.capacity - total;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    int *pairs = a.pairs + 2 * (int64_t)total;
    OutT *deltas = static_cast<OutT *>(a.deltas) + 3 * (int64_t)total;
    OutT *dists = static_cast<OutT *>(a.dists) + total;
    for (int64_t i = tid; i < 2 * rows; i += stride) pairs[i] = -1;
    for (int64_t i = tid; i < 3 * rows; i += stride) deltas[i] = (OutT)0;
    for (int64_t i = tid; i < rows; i += stride) dists[i] = (OutT)0;
}

__global__ void k_f32_to_f64(const float *__restrict__ src, double *__restrict__ dst, int64_t n)
{
    NNP_PDL_SYNC();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = (double)src[i];
}

__global__ void k_pullback(const int *__restrict__ pairs, const double *__restrict__ deltas,
                           const double *__restrict__ dists, const double *__restrict__ g, int count,
                           double *__restrict__ grad, int *__restrict__ flag)
{
    NNP_PDL_SYNC();
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    int i = pairs[2 * e], j = pairs[2 * e + 1];
    if (i == j || i < 0) return;
    double d = dists[e];
    if (d == 0.0) {
        atomicMin(flag, e + 1);  // first offending row, like the reference's report
        return;
    }
    double ge = g[e];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double c = ge * (deltas[3 * (size_t)e + k] / d);
        atomicAdd(&grad[3 * (size_t)i + k], c);
        atomicAdd(&grad[3 * (size_t)j + k], -c);
    }
}

constexpr int BOUNDS_BLOCKS = 128;

// accepted candidates kept per row between the two passes: 1.5x the mean row the capacity allows
int stage_width(const nnp_nl_params *p)
{
    int64_t w = (3 * (int64_t)p->capacity) / (2 * (int64_t)p->n_atoms) + 8;
    return (int)std::min<int64_t>(std::max<int64_t>(w, 16), NL_MAXROW);
}

size_t carve(NlArgs &a, const nnp_nl_params *p, void *ws)
{
    NnpArena ar(ws);
    const size_t n = (size_t)p->n_atoms;
    const size_t mc = (size_t)(p->max_cells > 0 ? p->max_cells : 1);
    a.cell_id = ar.take<int>(n);
    a.cell_start = ar.take<int>(mc + 1);
    a.cell_cursor = ar.take<int>(mc);
    a.tmp_order = ar.take<int>(n);
    a.sidx = ar.take<int>(n);
    a.rank_of = ar.take<int>(n);
    a.sbatch = ar.take<int>(n);
    a.row_count = ar.take<int>(n + 1 + nnp_scan_temp_ints((int64_t)std::max(n, mc) + 1));
    a.sample_ptr = ar.take<int>((size_t)p->n_samples + 1);
    a.scratch_col = ar.take<int>((size_t)p->capacity);
    a.scratch_t = ar.take<int>((size_t)p->capacity);
    a.stage_w = stage_width(p);
    a.stage_t = ar.take<int>(n * (size_t)a.stage_w);
    a.spos = ar.take<double>(3 * n);
    a.slpos = ar.take<float4>(n);
    a.scell = ar.take<int4>(n);
    a.bounds_partial = ar.take<double>(6 * BOUNDS_BLOCKS);
    a.grid = ar.take<GridDev>(1);
    return ar.bytes();
}

int validate(const nnp_nl_params *p)
{
    NNP_CHECK_ARG(p != nullptr, "params is NULL");
    NNP_CHECK_ARG(p->n_atoms >= 1, "n_atoms must be >= 1");
    NNP_CHECK_ARG(p->n_samples >= 1, "n_samples must be >= 1");
    NNP_CHECK_ARG(p->capacity >= 1, "capacity must be >= 1");
    NNP_CHECK_ARG(p->cutoff_lower >= 0.0 && p->cutoff_lower < p->cutoff_upper,
                  "cutoffs must satisfy 0 <= cutoff_lower < cutoff_upper");
    NNP_CHECK_ARG(p->box_kind >= 0 && p->box_kind <= 2, "unknown box kind");
    NNP_CHECK_ARG(p->strategy == NNP_STRATEGY_BRUTE || p->strategy == NNP_STRATEGY_CELL,
                  "strategy must be brute or cell");
    if (p->strategy == NNP_STRATEGY_CELL) {
        NNP_CHECK_ARG(p->max_cells >= 1, "max_cells must be >= 1 for the cell strategy");
        if (p->box_kind != NNP_BOX_NONE) {
            NNP_CHECK_ARG(p->grid_dims[0] >= 3 && p->grid_dims[1] >= 3 && p->grid_dims[2] >= 3,
                          "periodic cell grid needs >= 3 cells per axis");
            NNP_CHECK_ARG((int64_t)p->grid_dims[0] * p->grid_dims[1] * p->grid_dims[2] <=
                              (int64_t)p->max_cells,
                          "grid_dims exceed max_cells");
        }
    }
    if (p->box_kind != NNP_BOX_NONE)
        NNP_CHECK_ARG(p->box[0] > 0 && p->box[4] > 0 && p->box[8] > 0,
                      "box diagonal must be positive");
    return NNP_OK;
}

}  // namespace

extern "C" int nnp_nl_workspace_bytes(const nnp_nl_params *p, size_t *bytes)
{
    int rc = validate(p);
    if (rc) return rc;
    NNP_CHECK_ARG(bytes != nullptr, "bytes is NULL");
    NlArgs a{};
    *bytes = carve(a, p, nullptr);
    return NNP_OK;
}

extern "C" int nnp_nl_build(const nnp_nl_params *p, const double *pos, const int32_t *batch,
                            int32_t *pairs, void *deltas, void *dists, int32_t *row_ptr,
                            int32_t *order, int32_t *counts, void *workspace,
                            size_t workspace_bytes, nnp_stream_t stream_)
{
    int rc = validate(p);
    if (rc) return rc;
    NNP_CHECK_ARG(pos && batch && pairs && deltas && dists && counts && workspace,
                  "NULL buffer passed to nnp_nl_build");
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    NlArgs a{};
    size_t need = carve(a, p, workspace);
    if (need > workspace_bytes) {
        nnp_set_error("workspace too small: need %zu bytes, got %zu", need, workspace_bytes);
        return NNP_ERR_WORKSPACE;
    }
    a.n = p->n_atoms;
    a.n_samples = p->n_samples;
    a.capacity = p->capacity;
    a.strategy = p->strategy;
    a.flags = p->flags;
    a.periodic = p->box_kind != NNP_BOX_NONE;
    a.max_cells = p->max_cells > 0 ? p->max_cells : 1;
    a.cutoff = p->cutoff_upper;
    for (int k = 0; k < 9; ++k) a.inv_box[k] = p->inv_box[k];
    for (int k = 0; k < 3; ++k) a.host_dims[k] = p->grid_dims[k];
    Metric &m = a.metric;
    m.wrapped = a.periodic;
    m.lo2 = p->cutoff_lower * p->cutoff_lower;
    m.hi2 = p->cutoff_upper * p->cutoff_upper;
    if (a.periodic) {
        m.b00 = p->box[0];
        m.b10 = p->box[3];
        m.b11 = p->box[4];
        m.b20 = p->box[6];
        m.b21 = p->box[7];
        m.b22 = p->box[8];
        m.i00 = 1.0 / m.b00;
        m.i11 = 1.0 / m.b11;
        m.i22 = 1.0 / m.b22;
    }
    {
        // prefilter window: relative error of the float32 squared distance.  Differences enter
        // exact to 1 ulp(float); the periodic reduction adds ~ulp(box length) per component.
        double span = 0.0;
        if (a.periodic)
            for (int k = 0; k < 9; ++k) span = std::max(span, std::fabs(p->box[k]));
        const double eps = 32.0 * 1.1920929e-7 * (1.0 + 3.0 * span / p->cutoff_upper);
        MetricF &f = a.mf;
        f.b00 = (float)m.b00; f.b10 = (float)m.b10; f.b11 = (float)m.b11;
        f.b20 = (float)m.b20; f.b21 = (float)m.b21; f.b22 = (float)m.b22;
        f.i00 = (float)m.i00; f.i11 = (float)m.i11; f.i22 = (float)m.i22;
        f.hi2p = (float)(m.hi2 * (1.0 + eps)) * 1.000001f;
        f.lo2m = m.lo2 > 0.0 ? (float)(m.lo2 * (1.0 - eps)) * 0.999999f : -1.0f;
    }
    a.pos = pos;
    a.batch = batch;
    a.pairs = pairs;
    a.deltas = deltas;
    a.dists = dists;
    a.row_ptr = row_ptr ? row_ptr : a.row_count;
    a.order = order;
    a.counts = counts;
    int *scan_temp = a.row_count + a.n + 1;

    const int n = a.n;
    const int nb = nnp_blocks(n, 256);
    { NNP_PROF("k_sample_ptr", stream); nnp_launch((k_sample_ptr), NNP_GRID(nnp_blocks(a.n_samples + 1, 256)), 256, 0, stream, batch, n, a.n_samples, a.sample_ptr, counts); }

    if (a.strategy == NNP_STRATEGY_CELL) {
        int n_partial = 1;
        if (!a.periodic) {
            n_partial = std::min(BOUNDS_BLOCKS, nb);
            { NNP_PROF("k_bounds_partial", stream); nnp_launch((k_bounds_partial), NNP_GRID(n_partial), NL_THREADS, 0, stream, pos, n, a.bounds_partial); }
        }
        { NNP_PROF("k_grid_setup", stream); nnp_launch((k_grid_setup), NNP_GRID(1), 32, 0, stream, a, n_partial); }
        // cell_start (max_cells + 1 ints) and cell_cursor (max_cells ints) are carved back to back
        cudaMemsetAsync(a.cell_start, 0, (size_t)((char *)(a.cell_cursor + a.max_cells) - (char *)a.cell_start), stream);
        { NNP_PROF("k_cell_assign", stream); nnp_launch((k_cell_assign), NNP_GRID(nb), 256, 0, stream, a); }
        {
            NNP_PROF("scan_cells", stream);
            rc = nnp_exclusive_scan_i32(a.cell_start, a.cell_start, (int64_t)a.max_cells + 1,
                                        scan_temp, stream);
        }
        if (rc) return rc;
        { NNP_PROF("k_cell_scatter", stream); nnp_launch((k_cell_scatter), NNP_GRID(nb), 256, 0, stream, a); }
        { NNP_PROF("k_cell_rank", stream); nnp_launch((k_cell_rank), NNP_GRID(nb), 256, 0, stream, a); }
    } else {
        { NNP_PROF("k_identity_order", stream); nnp_launch((k_identity_order), NNP_GRID(nb), 256, 0, stream, a); }
    }
    NNP_CHECK_LAUNCH("neighbor binning");

    const int row_blocks = nnp_blocks(n, NL_WARPS);
    const bool f32 = p->flags & NNP_NL_F32_OUT;
    { NNP_PROF("k_rows_count", stream); nnp_launch((k_rows<false, double>), NNP_GRID(row_blocks), NL_THREADS, 0, stream, a); }
    {
        NNP_PROF("scan_rows", stream);
        rc = nnp_exclusive_scan_i32(a.row_count, a.row_ptr, (int64_t)n + 1, scan_temp, stream);
    }
    if (rc) return rc;
    if (f32)
        { NNP_PROF("k_rows_fill", stream); nnp_launch((k_rows<true, float>), NNP_GRID(row_blocks), NL_THREADS, 0, stream, a); }
    else
        { NNP_PROF("k_rows_fill", stream); nnp_launch((k_rows<true, double>), NNP_GRID(row_blocks), NL_THREADS, 0, stream, a); }
    if (!(p->flags & NNP_NL_NO_PAD)) {
        if (f32)
            { NNP_PROF("k_pad_tail", stream); nnp_launch((k_pad_tail<float>), NNP_GRID(std::min(nnp_blocks(a.capacity, 256), 148 * 8)), 256, 0, stream, a); }
        else
            { NNP_PROF("k_pad_tail", stream); nnp_launch((k_pad_tail<double>), NNP_GRID(std::min(nnp_blocks(a.capacity, 256), 148 * 8)), 256, 0, stream, a); }
    }
    NNP_CHECK_LAUNCH("neighbor rows");
    return NNP_OK;
}

extern "C" int nnp_f32_to_f64(const float *src, double *dst, int64_t n, nnp_stream_t stream)
{
    NNP_CHECK_ARG(src && dst && n >= 0, "bad arguments to nnp_f32_to_f64");
    if (n == 0) return NNP_OK;
    nnp_launch((k_f32_to_f64), NNP_GRID(nnp_blocks(n, 256)), 256, 0, static_cast<cudaStream_t>(stream), src, dst, n);
    NNP_CHECK_LAUNCH("f32_to_f64");
    return NNP_OK;
}

// Directional derivative of the pullback along a position tangent (neighbors.py:358-380): per edge
// the pair Hessian (1 - u u^T)/d applied to t_i - t_j, scattered +/- like the pullback itself, and
// the distance tangent u . (t_i - t_j) (zero on loops; the caller pre-zeroes the sentinel tail).
// Operation order as the reference: tdiff, ddot = sum_k u_k tdiff_k (left to right),
// hvp_k = g * (tdiff_k - u_k * ddot) / d.
__global__ void k_pullback_second(const int *__restrict__ pairs, const double *__restrict__ deltas,
                                  const double *__restrict__ dists, const double *__restrict__ g,
                                  const double *__restrict__ tangent, int count, double *__restrict__ grad,
                                  double *__restrict__ dtan, int *__restrict__ flag)
{
    NNP_PDL_SYNC();
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    int i = pairs[2 * e], j = pairs[2 * e + 1];
    if (i < 0) return;
    if (i == j) {
        dtan[e] = 0.0;
        return;
    }
    double d = dists[e];
    if (d == 0.0) {
        atomicMin(flag, e + 1);
        return;
    }
    double u[3], td[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        u[k] = deltas[3 * (size_t)e + k] / d;
        td[k] = __dsub_rn(tangent[3 * (size_t)i + k], tangent[3 * (size_t)j + k]);
    }
    const double ddot = __dadd_rn(__dadd_rn(__dmul_rn(u[0], td[0]), __dmul_rn(u[1], td[1])), __dmul_rn(u[2], td[2]));
    dtan[e] = ddot;
    const double ge = g[e];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double c = __dmul_rn(ge, __dsub_rn(td[k], __dmul_rn(u[k], ddot))) / d;
        atomicAdd(&grad[3 * (size_t)i + k], c);
        atomicAdd(&grad[3 * (size_t)j + k], -c);
    }
}

extern "C" int nnp_distance_pullback_second(const int32_t *pairs, const double *deltas, const double *dists,
                                            const double *g, const double *tangent, int32_t count,
                                            int32_t capacity, int32_t n_atoms, double *grad,
                                            double *distance_tangent, int32_t *flag_out, nnp_stream_t stream_)
{
    NNP_CHECK_ARG(grad && distance_tangent && flag_out && tangent && count >= 0 && capacity >= count && n_atoms >= 1,
                  "bad arguments to nnp_distance_pullback_second");
    NNP_CHECK_ARG(count == 0 || (pairs && deltas && dists && g),
                  "NULL edge buffer passed to nnp_distance_pullback_second");
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    cudaMemsetAsync(grad, 0, 3 * (size_t)n_atoms * sizeof(double), stream);
    cudaMemsetAsync(distance_tangent, 0, (size_t)capacity * sizeof(double), stream);
    cudaMemsetAsync(flag_out, 0x7f, sizeof(int), stream);
    if (count > 0)
        nnp_launch((k_pullback_second), NNP_GRID(nnp_blocks(count, 256)), 256, 0, stream, pairs, deltas, dists, g,
                   tangent, count, grad, distance_tangent, flag_out);
    NNP_CHECK_LAUNCH("distance_pullback_second");
    return NNP_OK;
}

extern "C" int nnp_distance_pullback(const int32_t *pairs, const double *deltas,
                                     const double *dists, const double *g, int32_t count,
                                     int32_t n_atoms, double *grad, int32_t *flag_out,
                                     nnp_stream_t stream_)
{
    NNP_CHECK_ARG(grad && flag_out && count >= 0 && n_atoms >= 1,
                  "bad arguments to nnp_distance_pullback");
    NNP_CHECK_ARG(count == 0 || (pairs && deltas && dists && g),
                  "NULL edge buffer passed to nnp_distance_pullback");
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    cudaMemsetAsync(grad, 0, 3 * (size_t)n_atoms * sizeof(double), stream);
    cudaMemsetAsync(flag_out, 0x7f, sizeof(int), stream);  // 0x7f7f7f7f = none
    if (count > 0)
        nnp_launch((k_pullback), NNP_GRID(nnp_blocks(count, 256)), 256, 0, stream, pairs, deltas, dists, g, count, grad,
                                                              flag_out);
    NNP_CHECK_LAUNCH("distance_pullback");
    return NNP_OK;
}
