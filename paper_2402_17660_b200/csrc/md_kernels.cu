// Langevin dynamics in the middle-thermostat splitting, one kernel per step on the device.
//
// Replaces langevin_middle_step (md.py:114-145): kick, half drift, Ornstein-Uhlenbeck velocity
// mixing, half drift.  State (positions, velocities) is float64 like the reference; the forces
// are the float32 output of the TensorNet step.  Every product and sum is rounded separately
// (__dmul_rn / __dadd_rn, no FMA contraction) in the reference's operation order, so with the
// same forces and the same noise the new state is bit-identical to the NumPy statement.
// The noise is either supplied by the caller (the reference's own Philox/ziggurat stream, for the
// drop-in step) or drawn on the device from Philox4x32-10 keyed by (seed, step, atom) with
// Box-Muller, so that a captured graph advances the stream by itself.
#include "nnp_common.cuh"

namespace {

struct Philox {
    uint32_t c[4];
    uint32_t k[2];
};

__device__ __forceinline__ void philox_round(Philox &p)
{
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t hi0 = __umulhi(M0, p.c[0]), lo0 = M0 * p.c[0];
    const uint32_t hi1 = __umulhi(M1, p.c[2]), lo1 = M1 * p.c[2];
    const uint32_t n0 = hi1 ^ p.c[1] ^ p.k[0], n1 = lo1, n2 = hi0 ^ p.c[3] ^ p.k[1], n3 = lo0;
    p.c[0] = n0;
    p.c[1] = n1;
    p.c[2] = n2;
    p.c[3] = n3;
}

// Philox4x32-10 (Salmon et al., SC'11): counter (c0..c3), key (k0, k1) -> four 32-bit words
__device__ __forceinline__ void philox4x32_10(Philox &p)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        philox_round(p);
        if (r < 9) {
            p.k[0] += 0x9E3779B9u;
            p.k[1] += 0xBB67AE85u;
        }
    }
}

// 64 random bits -> uniform double in (0, 1]
__device__ __forceinline__ double u01(uint32_t hi, uint32_t lo)
{
    const unsigned long long bits = ((unsigned long long)hi << 32 | lo) >> 11;   // 53 bits
    return ((double)bits + 1.0) * (1.0 / 9007199254740992.0);
}

__global__ void k_langevin_middle(double *__restrict__ pos, double *__restrict__ vel,
                                  const float *__restrict__ forces, const double *__restrict__ acc_scale,
                                  const double *__restrict__ sigma, const double *__restrict__ noise,
                                  unsigned long long seed, const unsigned long long *__restrict__ step_counter,
                                  double dt, double c1, double c2, float *__restrict__ pos32_out,
                                  int *__restrict__ flag, int n, const int *__restrict__ nl_counts,
                                  int nl_capacity)
{
    NNP_PDL_SYNC();
    // The neighbor structure overflowed in this step: the energy/forces kernels returned early and
    // `forces` still holds the previous step's values.  Freeze the state instead of integrating stale
    // forces (flag 2; the host regrows the list and resumes from here).
    if (nl_counts && nl_counts[0] > nl_capacity) {
        if (flag && blockIdx.x == 0 && threadIdx.x == 0) atomicMax(flag, 2);
        return;
    }
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double half_dt = 0.5 * dt;
    double xi[3] = {0.0, 0.0, 0.0};
    if (c2 > 0.0) {
        if (noise) {
            xi[0] = noise[3 * (size_t)i];
            xi[1] = noise[3 * (size_t)i + 1];
            xi[2] = noise[3 * (size_t)i + 2];
        } else {
            // two Philox blocks per atom and step: 8 words -> 4 uniforms -> 4 normals (3 used)
            const unsigned long long step = step_counter ? step_counter[0] : 0ull;
            double u[4];
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                Philox p;
                p.c[0] = (uint32_t)i;
                p.c[1] = (uint32_t)b;
                p.c[2] = (uint32_t)step;
                p.c[3] = (uint32_t)(step >> 32);
                p.k[0] = (uint32_t)seed;
                p.k[1] = (uint32_t)(seed >> 32);
                philox4x32_10(p);
                u[2 * b] = u01(p.c[0], p.c[1]);
                u[2 * b + 1] = u01(p.c[2], p.c[3]);
            }
            const double r0 = sqrt(-2.0 * log(u[0])), r1 = sqrt(-2.0 * log(u[2]));
            double s0, c0, s1, c1b;
            sincospi(2.0 * u[1], &s0, &c0);
            sincospi(2.0 * u[3], &s1, &c1b);
            xi[0] = r0 * c0;
            xi[1] = r0 * s0;
            xi[2] = r1 * c1b;
        }
    }
    const double a = acc_scale[i], sg = sigma[i];
    bool finite = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float f = forces[3 * (size_t)i + k];
        finite = finite && isfinite(f);
        // accel = forces * (FORCE_TO_ACCELERATION / m);  v = v + dt * accel
        double v = __dadd_rn(vel[3 * (size_t)i + k], __dmul_rn(dt, __dmul_rn((double)f, a)));
        // x = x + 0.5 * dt * v
        double x = __dadd_rn(pos[3 * (size_t)i + k], __dmul_rn(half_dt, v));
        // v = c1 * v + c2 * sigma * noise
        if (c2 > 0.0) v = __dadd_rn(__dmul_rn(c1, v), __dmul_rn(__dmul_rn(c2, sg), xi[k]));
        x = __dadd_rn(x, __dmul_rn(half_dt, v));
        vel[3 * (size_t)i + k] = v;
        pos[3 * (size_t)i + k] = x;
        if (pos32_out) pos32_out[3 * (size_t)i + k] = (float)x;
    }
    if (!finite && flag) atomicMax(flag, 1);
}

__global__ void k_advance_counter(unsigned long long *counter, const int *__restrict__ nl_counts, int nl_capacity)
{
    NNP_PDL_SYNC();
    if (nl_counts && nl_counts[0] > nl_capacity) return;     // frozen step: the random stream does not advance
    counter[0] += 1ull;
}

}  // namespace

extern "C" int nnp_md_langevin_middle(double *pos, double *vel, const float *forces, const double *acc_scale,
                                      const double *sigma, const double *noise, uint64_t seed,
                                      uint64_t *step_counter, double dt, double c1, double c2,
                                      float *pos32_out, int32_t *nonfinite_flag, int32_t n,
                                      const int32_t *nl_counts, int32_t nl_capacity, nnp_stream_t stream)
{
    NNP_CHECK_ARG(pos && vel && forces && acc_scale && sigma && n >= 1, "bad arguments to nnp_md_langevin_middle");
    NNP_CHECK_ARG(dt > 0.0 && c1 >= 0.0 && c1 <= 1.0 && c2 >= 0.0, "bad integrator coefficients");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    nnp_launch((k_langevin_middle), NNP_GRID(nnp_blocks(n, 256)), 256, 0, st, 
        pos, vel, forces, acc_scale, sigma, noise, (unsigned long long)seed,
        reinterpret_cast<const unsigned long long *>(step_counter), dt, c1, c2, pos32_out, nonfinite_flag, n,
        nl_counts, nl_capacity);
    if (step_counter)
        nnp_launch((k_advance_counter), NNP_GRID(1), 1, 0, st, reinterpret_cast<unsigned long long *>(step_counter),
                   nl_counts, nl_capacity);
    NNP_CHECK_LAUNCH("langevin_middle");
    return NNP_OK;
}
