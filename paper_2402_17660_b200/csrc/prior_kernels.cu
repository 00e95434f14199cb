// Analytic pair priors (switched Coulomb, ZBL screened repulsion, D2 dispersion) on a device
// neighbor list, float64 throughout.
//
// Replaces the pair functions of priors.py:139-148 (Coulomb), :170-185 (ZBL), :222-245 (D2) and
// the assembly of priors.py:61-88: every undirected pair contributes half of its energy to each
// endpoint and equal and opposite forces along the minimum-image direction.  One thread per list
// row; a full (directed) list is reduced to its half by keeping rows with i < j, self loops are
// skipped.  The enabled terms are evaluated in one pass over the pair.  Per-atom sums use float64
// atomics (their order is the only difference to the NumPy statement: ~1e-16 relative).
#include "nnp_common.cuh"

namespace {

__device__ __forceinline__ void cosine_envelope(double d, double ru, double &env, double &denv)
{
    // radial.py:11-39 with cutoff_lower = 0 (operation order of the reference)
    const double phase = 3.141592653589793 * d / ru;
    const bool in = d <= ru;
    env = in ? 0.5 * (cos(phase) + 1.0) : 0.0;
    denv = in ? -0.5 * 3.141592653589793 / ru * sin(phase) : 0.0;
}

__global__ void k_prior_pairs(nnp_prior_params p, const int *__restrict__ pairs,
                              const double *__restrict__ deltas, const double *__restrict__ dists,
                              const int *__restrict__ count_dev, int count_host, int full_list,
                              const double *__restrict__ charge, const double *__restrict__ znum,
                              const double *__restrict__ zpow, const double *__restrict__ c6,
                              const double *__restrict__ rvdw, double *__restrict__ per_atom,
                              double *__restrict__ forces)
{
    NNP_PDL_SYNC();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int count = count_dev ? count_dev[0] : count_host;
    if (r >= count) return;
    const int i = pairs[2 * (size_t)r], j = pairs[2 * (size_t)r + 1];
    if (i < 0 || i == j || (full_list && i > j)) return;
    const double d = dists[r];
    double e = 0.0, de = 0.0;
    if (p.flags & NNP_PRIOR_COULOMB) {
        const double qq = p.coulomb_constant * charge[i] * charge[j];
        const bool inside = d < p.switch_radius;
        const double phase = 3.141592653589793 * d / p.switch_radius;
        const double sw = inside ? 0.5 * (1.0 - cos(phase)) : 1.0;
        const double dsw = inside ? 0.5 * 3.141592653589793 / p.switch_radius * sin(phase) : 0.0;
        e += qq * sw / d;
        de += qq * (dsw / d - sw / (d * d));
    }
    if (p.flags & (NNP_PRIOR_ZBL | NNP_PRIOR_D2)) {
        double env, denv;
        cosine_envelope(d, p.cutoff_upper, env, denv);
        if (p.flags & NNP_PRIOR_ZBL) {
            const double a = p.zbl_prefactor / (zpow[i] + zpow[j]);
            const double x = d / a;
            const double ck[4] = {0.18175, 0.50986, 0.28022, 0.02817};
            const double ek[4] = {3.19980, 0.94229, 0.40290, 0.20162};
            double screen = 0.0, dscreen = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double t = ck[k] * exp(-ek[k] * x);
                screen += t;
                dscreen += t * ek[k];
            }
            dscreen = -dscreen / a;
            const double bare = p.coulomb_constant * znum[i] * znum[j] / d;
            e += bare * screen * env;
            de += -bare / d * screen * env + bare * dscreen * env + bare * screen * denv;
        }
        if (p.flags & NNP_PRIOR_D2) {
            const double cc = sqrt(c6[i] * c6[j]);
            const double rsum = rvdw[i] + rvdw[j];
            const double arg = p.d2_steep * (d / rsum - 1.0);
            double damp;
            if (arg >= 0.0) {
                damp = 1.0 / (1.0 + exp(-arg));
            } else {
                const double ex = exp(arg);
                damp = ex / (1.0 + ex);
            }
            const double ddamp = damp * (1.0 - damp) * p.d2_steep / rsum;
            const double inv6 = pow(d, -6.0);
            e += -p.d2_s6 * cc * inv6 * damp * env;
            de += -p.d2_s6 * cc * (-6.0 * inv6 / d * damp * env + inv6 * ddamp * env + inv6 * damp * denv);
        }
    }
    atomicAdd(per_atom + i, 0.5 * e);
    atomicAdd(per_atom + j, 0.5 * e);
    if (forces) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double pf = -de * (deltas[3 * (size_t)r + k] / d);
            atomicAdd(forces + 3 * (size_t)i + k, pf);
            atomicAdd(forces + 3 * (size_t)j + k, -pf);
        }
    }
}

}  // namespace

extern "C" int nnp_priors_pair_terms(const nnp_prior_params *p, const int32_t *pairs, const double *deltas,
                                     const double *dists, const int32_t *count_dev, int32_t count_host,
                                     int32_t full_list, const double *charge, const double *znum,
                                     const double *zpow, const double *c6, const double *rvdw,
                                     int32_t n_atoms, double *per_atom, double *forces, nnp_stream_t stream)
{
    NNP_CHECK_ARG(p && pairs && deltas && dists && per_atom && n_atoms >= 1 && count_host >= 0,
                  "bad arguments to nnp_priors_pair_terms");
    NNP_CHECK_ARG(!(p->flags & NNP_PRIOR_COULOMB) || (charge && p->switch_radius > 0.0),
                  "the Coulomb term needs charges and a positive switch radius");
    NNP_CHECK_ARG(!(p->flags & NNP_PRIOR_ZBL) || (znum && zpow), "the ZBL term needs atomic numbers");
    NNP_CHECK_ARG(!(p->flags & NNP_PRIOR_D2) || (c6 && rvdw && p->d2_s6 > 0.0),
                  "the dispersion term needs C6 coefficients and radii");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaMemsetAsync(per_atom, 0, sizeof(double) * (size_t)n_atoms, st);
    if (forces) cudaMemsetAsync(forces, 0, sizeof(double) * 3 * (size_t)n_atoms, st);
    if (count_host > 0)
        nnp_launch((k_prior_pairs), NNP_GRID(nnp_blocks(count_host, 256)), 256, 0, st, 
            *p, pairs, deltas, dists, count_dev, count_host, full_list, charge, znum, zpow, c6, rvdw, per_atom,
            forces);
    NNP_CHECK_LAUNCH("prior_pairs");
    return NNP_OK;
}
