/*
 * oracle/nl_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Plain-C, serial, float64 restatement of the reference's half-list pair
 * enumeration (the only natively-compiled code of the reference):
 *   pkg/src/nnpkit/_neighbor_kernels.py:24-51    brute, open boundaries
 *   pkg/src/nnpkit/_neighbor_kernels.py:55-96    brute, staircase minimum image
 *   pkg/src/nnpkit/_neighbor_kernels.py:100-149  cell scan, clamped 27 cells
 *   pkg/src/nnpkit/_neighbor_kernels.py:153-233  cell scan, periodic 27 cells
 * and of the cell binning that feeds them:
 *   pkg/src/nnpkit/neighbors.py:127-133          stable sort of atoms by flat cell id
 *
 * The four reference kernels differ only in (a) where candidates j come from
 * and (b) whether the displacement is wrapped, so they are restated here as one
 * enumeration routine with two switches.  Arithmetic order is the reference's:
 * d = r_i - r_j with i < j, wrap c then b then a with rint(component/diagonal),
 * d2 = (dx*dx + dy*dy) + dz*dz, window lo2 < d2 <= hi2 on SQUARED distances,
 * counting continues past capacity.  Build with -ffp-contract=off so no FMA is
 * formed (numba without fastmath does not contract either); see oracle/Makefile.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int wrapped;              /* 0: open, 1: staircase minimum image */
    double b00, b10, b11, b20, b21, b22;
    double lo2, hi2;
} nlo_metric;

/* Displacement r_i - r_j (i < j) reduced c -> b -> a; returns squared norm. */
static inline double nlo_delta(const nlo_metric *m, const double *pi, const double *pj,
                               double *out)
{
    double dx = pi[0] - pj[0];
    double dy = pi[1] - pj[1];
    double dz = pi[2] - pj[2];
    if (m->wrapped) {
        double s = rint(dz / m->b22);
        dx -= s * m->b20;
        dy -= s * m->b21;
        dz -= s * m->b22;
        s = rint(dy / m->b11);
        dx -= s * m->b10;
        dy -= s * m->b11;
        dx -= m->b00 * rint(dx / m->b00);
    }
    out[0] = dx;
    out[1] = dy;
    out[2] = dz;
    return dx * dx + dy * dy + dz * dz;
}

static inline void nlo_emit(int64_t *count, int64_t capacity, int64_t i, int64_t j,
                            const double *d, double d2, int64_t *pairs, double *deltas,
                            double *dists)
{
    int64_t c = *count;
    if (c < capacity) {
        pairs[2 * c] = i;
        pairs[2 * c + 1] = j;
        deltas[3 * c] = d[0];
        deltas[3 * c + 1] = d[1];
        deltas[3 * c + 2] = d[2];
        dists[c] = sqrt(d2);
    }
    *count = c + 1;
}

static void nlo_fill_metric(nlo_metric *m, const double *box9, double r_lower, double r_upper)
{
    memset(m, 0, sizeof(*m));
    m->lo2 = r_lower * r_lower;
    m->hi2 = r_upper * r_upper;
    if (box9) {
        m->wrapped = 1;
        m->b00 = box9[0];
        m->b10 = box9[3];
        m->b11 = box9[4];
        m->b20 = box9[6];
        m->b21 = box9[7];
        m->b22 = box9[8];
    }
}

/*
 * All-pairs enumeration, rows i ascending, j = i+1..n-1 ascending.
 * box9 == NULL selects open boundaries.  Returns the number of pairs found
 * (may exceed capacity).
 */
int64_t nlo_brute_half(const double *pos, const int64_t *batch, int64_t n, const double *box9,
                       double r_lower, double r_upper, int64_t capacity, int64_t *pairs,
                       double *deltas, double *dists)
{
    nlo_metric m;
    nlo_fill_metric(&m, box9, r_lower, r_upper);
    int64_t count = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double *pi = pos + 3 * i;
        int64_t bi = batch[i];
        for (int64_t j = i + 1; j < n; ++j) {
            if (batch[j] != bi)
                continue;
            double d[3];
            double d2 = nlo_delta(&m, pi, pos + 3 * j, d);
            if (d2 > m.lo2 && d2 <= m.hi2)
                nlo_emit(&count, capacity, i, j, d, d2, pairs, deltas, dists);
        }
    }
    return count;
}

/*
 * Cell-list enumeration.  coords [n,3] are integer cell coordinates, dims[3]
 * the grid, order/start the atoms sorted by flat cell id (start has ncell+1
 * entries).  periodic != 0 wraps neighbour cells (the grid then has >= 3
 * cells per axis, neighbors.py:107-109), otherwise out-of-range cells are
 * skipped.  Emission order is the reference's: atom i ascending, offsets
 * (-1,0,1)^3 with the last axis fastest, then cell order; candidates with
 * j <= i are skipped so every unordered pair appears once.
 */
int64_t nlo_cell_half(const double *pos, const int64_t *batch, int64_t n, const double *box9,
                      int periodic, double r_lower, double r_upper, const int64_t *coords,
                      const int64_t *dims, const int64_t *order, const int64_t *start,
                      int64_t capacity, int64_t *pairs, double *deltas, double *dists)
{
    nlo_metric m;
    nlo_fill_metric(&m, box9, r_lower, r_upper);
    const int64_t m0 = dims[0], m1 = dims[1], m2 = dims[2];
    int64_t count = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double *pi = pos + 3 * i;
        int64_t bi = batch[i];
        for (int o0 = -1; o0 <= 1; ++o0) {
            int64_t n0 = coords[3 * i] + o0;
            if (periodic) {
                n0 = n0 < 0 ? n0 + m0 : (n0 >= m0 ? n0 - m0 : n0);
            } else if (n0 < 0 || n0 >= m0) {
                continue;
            }
            for (int o1 = -1; o1 <= 1; ++o1) {
                int64_t n1 = coords[3 * i + 1] + o1;
                if (periodic) {
                    n1 = n1 < 0 ? n1 + m1 : (n1 >= m1 ? n1 - m1 : n1);
                } else if (n1 < 0 || n1 >= m1) {
                    continue;
                }
                for (int o2 = -1; o2 <= 1; ++o2) {
                    int64_t n2 = coords[3 * i + 2] + o2;
                    if (periodic) {
                        n2 = n2 < 0 ? n2 + m2 : (n2 >= m2 ? n2 - m2 : n2);
                    } else if (n2 < 0 || n2 >= m2) {
                        continue;
                    }
                    int64_t flat = (n0 * m1 + n1) * m2 + n2;
                    for (int64_t p = start[flat]; p < start[flat + 1]; ++p) {
                        int64_t j = order[p];
                        if (j <= i || batch[j] != bi)
                            continue;
                        double d[3];
                        double d2 = nlo_delta(&m, pi, pos + 3 * j, d);
                        if (d2 > m.lo2 && d2 <= m.hi2)
                            nlo_emit(&count, capacity, i, j, d, d2, pairs, deltas, dists);
                    }
                }
            }
        }
    }
    return count;
}

/*
 * Stable counting sort of atoms by flat cell id (neighbors.py:127-133 uses a
 * stable argsort + bincount + cumsum; the result is identical).
 */
void nlo_sort_cells(const int64_t *coords, const int64_t *dims, int64_t n, int64_t *order,
                    int64_t *start /* ncell + 1 */)
{
    const int64_t ncell = dims[0] * dims[1] * dims[2];
    memset(start, 0, (size_t)(ncell + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        int64_t flat = (coords[3 * i] * dims[1] + coords[3 * i + 1]) * dims[2] + coords[3 * i + 2];
        start[flat + 1] += 1;
    }
    for (int64_t c = 0; c < ncell; ++c)
        start[c + 1] += start[c];
    int64_t *cursor = (int64_t *)malloc((size_t)(ncell > 0 ? ncell : 1) * sizeof(int64_t));
    memcpy(cursor, start, (size_t)ncell * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        int64_t flat = (coords[3 * i] * dims[1] + coords[3 * i + 1]) * dims[2] + coords[3 * i + 2];
        order[cursor[flat]++] = i;
    }
    free(cursor);
}
