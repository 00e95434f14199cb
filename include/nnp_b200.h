/*
 * nnp_b200.h -- C ABI of the B200-native neighbor search + TensorNet energy/forces step.
 *
 * This is the drop-in boundary for the hot path of the reference package `nnpkit`
 * (/root/reference/pkg/src/nnpkit).  Every entry point cites the reference interface it
 * replaces.  Conventions shared by all calls:
 *
 *  - plain pointers and sizes only; all array pointers are DEVICE pointers unless the
 *    name ends in `_host`;
 *  - the caller owns every buffer (inputs, outputs, workspace); nothing is allocated
 *    inside a call, so every call is CUDA-graph capturable ("static shapes
 *    and fixed memory addresses");
 *  - calls only enqueue work on `stream` and never synchronise;
 *  - return value 0 = success, negative = error code below; nnp_last_error() gives a
 *    thread-local message.  No C++ exception crosses this boundary;
 *  - data-dependent overflow is reported through device memory (`counts`), mirroring
 *    CapacityError.required (errors.py:32-45, neighbors.py:204-207): kernels keep
 *    counting past capacity (_neighbor_kernels.py:43-50) and the host wrapper raises.
 */
#ifndef NNP_B200_H
#define NNP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *nnp_stream_t; /* a cudaStream_t */

#define NNP_OK 0
#define NNP_ERR_INVALID (-1)   /* bad argument (host-detectable ValidationError) */
#define NNP_ERR_WORKSPACE (-2) /* workspace too small */
#define NNP_ERR_CUDA (-3)      /* a CUDA runtime call failed */
#define NNP_ERR_UNSUPPORTED (-4)

/* box kinds: _neighbor_kernels.py:18-20 */
#define NNP_BOX_NONE 0
#define NNP_BOX_ORTHORHOMBIC 1
#define NNP_BOX_TRICLINIC 2

/* strategies after host-side resolution of "auto" (neighbors.py:155-157) */
#define NNP_STRATEGY_BRUTE 0
#define NNP_STRATEGY_CELL 1

/* flags */
#define NNP_NL_FULL_LIST 1  /* NeighborSpec.full_list (neighbors.py:43) */
#define NNP_NL_SELF_LOOPS 2 /* NeighborSpec.include_self_loops (neighbors.py:42) */
#define NNP_NL_RENUMBER 4   /* rows/cols in cell-sorted atom numbering (internal model path) */
#define NNP_NL_F32_OUT 8    /* deltas/distances written as float32 instead of float64 */
#define NNP_NL_NO_PAD 16    /* do not write -1/0 sentinels into the unused tail */
#define NNP_NL_UNSORTED 32  /* NeighborSpec.deterministic = False (neighbors.py:44,221): rows stay grouped by
                               receiver (row_ptr is valid) but the order inside a row is unspecified */

const char *nnp_last_error(void);
int nnp_version(void);
/* sizeof of the ABI structs as this library was compiled (0 = nnp_nl_params, 1 = nnp_tn_model,
 * 2 = nnp_prior_params; -1 for anything else): lets a binding check its own struct layout. */
int nnp_abi_sizeof(int which);

/* ------------------------------------------------------------------ neighbor search
 * Replaces build_neighbor_list (neighbors.py:136-235) and the four numba kernels
 * (_neighbor_kernels.py:24-233), the grid construction (neighbors.py:103-124) and the cell
 * sort (neighbors.py:127-133).
 */
typedef struct nnp_nl_params {
    int32_t n_atoms;
    int32_t n_samples;    /* max(batch)+1 */
    int32_t capacity;     /* rows of the output arrays (NeighborSpec.capacity) */
    int32_t box_kind;     /* NNP_BOX_* */
    int32_t strategy;     /* NNP_STRATEGY_* */
    int32_t flags;        /* NNP_NL_* */
    int32_t grid_dims[3]; /* periodic cell grid floor(widths/cutoff), each >= 3 (host computed,
                             neighbors.py:103-109); ignored for open systems (device computed) */
    int32_t max_cells;    /* cells the workspace is sized for (open systems clamp to it) */
    double cutoff_lower, cutoff_upper;
    double box[9];        /* rows a,b,c, lower triangular (system.py:34-38) */
    double inv_box[9];    /* inverse of box (host computed, float64) */
} nnp_nl_params;

int nnp_nl_workspace_bytes(const nnp_nl_params *p, size_t *bytes);

/*
 * Outputs:
 *   pairs  [capacity,2] int32   (i, j); -1 in unused rows unless NNP_NL_NO_PAD
 *   deltas [capacity,3] float64 (float32 with NNP_NL_F32_OUT)  r_i - r_j, minimum image
 *   dists  [capacity]   same type
 *   row_ptr [n_atoms+1] int32 or NULL: CSR offsets of the (i, j)-sorted rows
 *   order   [n_atoms]   int32 or NULL: with NNP_NL_RENUMBER, order[s] = original index of
 *                                      the atom numbered s in the output (identity otherwise)
 *   counts  int32[4]: [0] rows required (directed pairs + loops; may exceed capacity, then
 *                     nothing is written), [1] longest row, [2] number of cells, [3] reserved
 * Rows come out sorted by (i, j) -- the reference's deterministic order (neighbors.py:221-225).
 * `pos` is float64 [n,3]; `batch` int32 [n], non-decreasing from 0 (system.py:231-235).
 */
int nnp_nl_build(const nnp_nl_params *p, const double *pos, const int32_t *batch, int32_t *pairs,
                 void *deltas, void *dists, int32_t *row_ptr, int32_t *order, int32_t *counts,
                 void *workspace, size_t workspace_bytes, nnp_stream_t stream);

/* float32 positions -> float64 (exact), so the model path tests the same bits as the oracle */
int nnp_f32_to_f64(const float *src, double *dst, int64_t n, nnp_stream_t stream);

/*
 * distance_pullback (neighbors.py:345-355): grad[i] += g_e * u_e, grad[j] -= g_e * u_e over
 * valid rows; self loops contribute nothing.  deltas/dists/g/grad are float64.  flag_out[0]
 * is 0x7f7f7f7f when all is well, else 1 + the first row holding a zero-distance non-loop pair
 * (NumericError, neighbors.py:333-338).
 */
int nnp_distance_pullback(const int32_t *pairs, const double *deltas, const double *dists,
                          const double *g, int32_t count, int32_t n_atoms, double *grad,
                          int32_t *flag_out, nnp_stream_t stream);

/*
 * distance_pullback_second (neighbors.py:358-380): directional derivative of the pullback along
 * a position tangent [n_atoms,3], with the analytic pair Hessian (1 - u u^T)/d per edge.
 *   grad [n_atoms,3] = sum_e +/- g_e (t_ij - u_e (u_e . t_ij)) / d_e,  t_ij = tangent[i] - tangent[j]
 *   distance_tangent [capacity] = u_e . t_ij on valid rows, 0 on loops and in sentinel slots.
 * All arrays float64; flag_out as in nnp_distance_pullback.
 */
int nnp_distance_pullback_second(const int32_t *pairs, const double *deltas, const double *dists,
                                 const double *g, const double *tangent, int32_t count,
                                 int32_t capacity, int32_t n_atoms, double *grad,
                                 double *distance_tangent, int32_t *flag_out, nnp_stream_t stream);

/* ------------------------------------------------------------------ TensorNet step
 * Replaces GraphPotential.evaluate (graphnet.py:567-580) = forward (graphnet.py:317-412) +
 * backward_forces (graphnet.py:516-537) with the TensorNet arithmetic of SURVEY.md
 * Appendix A.  Weights are float32 device arrays prepared by the host wrapper.
 */
#define NNP_TN_MAX_LAYERS 8

/* A GEMM weight W[N,K] (row-major float32 on the device).  The tensor-core kernels split it into
 * TF32 hi/lo parts themselves (once per CTA for the 128 x 128 channel mixes, whose weight lives in
 * tensor memory). */
typedef struct {
    const float *w;
} nnp_gemm_weight;

typedef struct nnp_tn_model {
    int32_t channels;  /* C: 32, 64 or 128 (GNConfig.embedding_dimension, graphnet.py:59) */
    int32_t num_rbf;   /* K (only used by the host when it builds the tables) */
    int32_t num_layers;
    int32_t max_z;
    int32_t num_knots; /* radial tables: cubic Hermite in u = exp(cutoff_lower - d) */
    float cutoff_lower, cutoff_upper;
    float u_min, u_step; /* knot k sits at u_min + k*u_step */
    float mean, std;     /* per-atom raw*std + mean (graphnet.py:406) */
    float h2_b;
    /* species tables: Z_e = z_recv[z_i] + z_send[z_j]  (emb2 bias folded into z_send) */
    const float *z_recv; /* [max_z, C] */
    const float *z_send; /* [max_z, C] */
    /* radial tables [(L+1)][num_knots][2][3][C]: table 0 = distance projections dp1..3 of the
       embedding, table 1+l = radial MLP of layer l (before the cosine envelope); per knot the
       values and the slopes (times u_step) that define the cubic Hermite interpolant in
       x = (u-u_k)/u_step on each knot interval */
    const float *tables;
    /* the same interpolants expanded per knot interval into monomial coefficients c0..c3 of
       x = (u-u_k)/u_step: [(L+1)][num_knots-1][4][3][C] (Horner form for the kernels that visit
       intervals in no particular order) */
    const float *tables_mono;
    const float *init_norm_g, *init_norm_b;             /* [C] */
    nnp_gemm_weight es0_w, es0_wT;                      /* [2C,C], [C,2C] */
    nnp_gemm_weight es1_w, es1_wT;                      /* [3C,2C], [2C,3C] */
    const float *es0_b, *es1_b;                         /* [2C], [3C] */
    nnp_gemm_weight et_w[3], et_wT[3];                  /* [C,C] each (I, A, S mixes) */
    nnp_gemm_weight layer_t_w[NNP_TN_MAX_LAYERS][6];    /* [C,C] each: lt0..lt5 */
    nnp_gemm_weight layer_t_wT[NNP_TN_MAX_LAYERS][6];   /* transposes (reverse sweep) */
    const float *out_norm_g, *out_norm_b;               /* [3C] */
    nnp_gemm_weight lin_w, lin_wT;                      /* [C,3C], [3C,C] */
    nnp_gemm_weight h1_w, h1_wT;                        /* [C/2,C], [C,C/2] */
    const float *lin_b, *h1_b;                          /* [C], [C/2] */
    const float *h2_w;                                  /* [C/2] */
    /* Embedding reverse by node-level projection (optional; embed_projection = 0 keeps the
       per-channel edge kernel).  The distance projections are linear in the expnorm basis,
       dp_j(rho)[c] = sum_k dp_wT[j][k][c] rho_k + dp_b[j][c], so dE/dX0 is first contracted over
       channels per node (two tcgen05 GEMMs against species-weighted copies of dp_wT, built on the
       device from the species present in the step) and every edge then costs 9 x num_rbf
       multiply-adds instead of ~60 per channel.  Needs num_rbf == 32; steps with more than four
       species fall back to the per-channel kernel on the device. */
    int32_t embed_projection;
    /* GEMM engine of this model's calls: 0 = the library default (nnp_set_gemm_mode), 5 = streaming
       tcgen05 mixes, 3 = per-tile tcgen05, 1 = mma.sync, 8 = FP32 FFMA.  Carried by the model so that
       concurrent callers (threads, devices) do not share a mode switch. */
    int32_t gemm_mode;
    const float *dp_wT;                                 /* [3][num_rbf][C] */
    const float *dp_b;                                  /* [3][C] */
    const float *rbf_means, *rbf_betas;                 /* [num_rbf] (radial.py:62-73) */
} nnp_tn_model;

int nnp_tn_workspace_bytes(const nnp_tn_model *m, int32_t n_atoms, int32_t capacity,
                           int32_t n_samples, size_t *bytes);

/*
 * One energy-and-forces evaluation on a prebuilt directed neighbor structure in CSR form
 * (full list with self loops, rows sorted by (i, j), as nnp_nl_build emits with
 * NNP_NL_FULL_LIST | NNP_NL_SELF_LOOPS | NNP_NL_F32_OUT).
 *   species [n] int32, batch [n] int32: in ORIGINAL atom order
 *   order   [n] int32 or NULL: atom numbering of the neighbor structure (see nnp_nl_build)
 *   row_ptr [n+1], pairs [capacity,2] int32, deltas [capacity,3] f32, dists [capacity] f32
 *   energy [n_samples] f32, forces [n,3] f32 (or NULL: energy only), per_atom [n] f32 or NULL;
 *   all three in original atom order.
 *   nl_counts: the int32[4] written by nnp_nl_build; if counts[0] > capacity the step writes
 *   nothing (the host raises CapacityError after the stream has drained).
 */
int nnp_tn_energy_forces(const nnp_tn_model *m, int32_t n_atoms, int32_t n_samples,
                         int32_t capacity, const int32_t *species, const int32_t *batch,
                         const int32_t *order, const int32_t *row_ptr, const int32_t *pairs,
                         const float *deltas, const float *dists, const int32_t *nl_counts,
                         float *energy, float *forces, float *per_atom, void *workspace,
                         size_t workspace_bytes, nnp_stream_t stream);

/* ------------------------------------------------------------------ MD integrator
 * Replaces langevin_middle_step (md.py:114-145): kick, half drift, Ornstein-Uhlenbeck velocity
 * mixing, half drift, in float64 with the reference's operation order (bit-identical to the NumPy
 * statement for equal forces and noise).
 *   pos, vel   [n,3] float64, updated in place       forces [n,3] float32 (the step's output)
 *   acc_scale  [n]   float64 = FORCE_TO_ACCELERATION / m_i (units.py:26)
 *   sigma      [n]   float64 = sqrt(k_B T FORCE_TO_ACCELERATION / m_i) (md.py:131-133)
 *   noise      [n,3] float64 standard normals supplied by the caller (the reference's own
 *              Philox stream), or NULL: drawn on the device from Philox4x32-10 keyed by
 *              (seed, *step_counter, atom) with Box-Muller
 *   step_counter device uint64 or NULL; incremented by the call, so a captured graph advances
 *              the random stream by itself
 *   c1 = exp(-gamma dt), c2 = sqrt(1 - c1^2) (md.py:128-129); c2 == 0 skips the mixing
 *   pos32_out  optional [n,3] float32 copy of the new positions
 *   nonfinite_flag optional device int32, set to 1 when a force is not finite (md.py:124-125) and to
 *              2 when the step was frozen because of a neighbor overflow
 *   nl_counts, nl_capacity: optional counts of the nnp_nl_build that fed this step; when
 *              nl_counts[0] > nl_capacity the forces are stale, so positions, velocities and the
 *              step counter are left untouched (the caller regrows the list and repeats the step)
 */
int nnp_md_langevin_middle(double *pos, double *vel, const float *forces, const double *acc_scale,
                           const double *sigma, const double *noise, uint64_t seed,
                           uint64_t *step_counter, double dt, double c1, double c2,
                           float *pos32_out, int32_t *nonfinite_flag, int32_t n,
                           const int32_t *nl_counts, int32_t nl_capacity, nnp_stream_t stream);

/* ------------------------------------------------------------------ analytic pair priors
 * Replaces the pair functions and the assembly of priors.py:61-88,139-148,170-185,222-245 on a
 * device neighbor list (float64 deltas / distances as nnp_nl_build writes them).  Every undirected
 * pair gives half of its energy to each endpoint and equal and opposite forces; a directed list is
 * reduced to rows with i < j, self loops are skipped.  Per-atom inputs are prepared by the host:
 *   charge [n] partial charges (Coulomb); znum [n] atomic numbers as float64 and zpow [n] = Z^0.23
 *   (ZBL); c6 [n] (eV A^6) and rvdw [n] (A) (D2).  per_atom [n] and forces [n,3] (may be NULL) are
 *   float64 and are zeroed by the call.  count_dev (device int32, e.g. the list's counts[0]) overrides
 *   count_host as the number of valid rows when not NULL; count_host then only sizes the launch. */
#define NNP_PRIOR_COULOMB 1
#define NNP_PRIOR_ZBL 2
#define NNP_PRIOR_D2 4
typedef struct nnp_prior_params {
    int32_t flags;            /* NNP_PRIOR_* */
    int32_t reserved;
    double cutoff_upper;      /* the list's cutoff: cosine envelope of ZBL and D2 (priors.py:176,229) */
    double coulomb_constant;  /* eV A / e^2 (units.py:13) */
    double switch_radius;     /* Coulomb short-range switch (priors.py:124) */
    double zbl_prefactor;     /* 0.8854 a0 (priors.py:44) */
    double d2_s6, d2_steep;   /* priors.py:200-201 */
} nnp_prior_params;
int nnp_priors_pair_terms(const nnp_prior_params *p, const int32_t *pairs, const double *deltas,
                          const double *dists, const int32_t *count_dev, int32_t count_host,
                          int32_t full_list, const double *charge, const double *znum, const double *zpow,
                          const double *c6, const double *rvdw, int32_t n_atoms, double *per_atom,
                          double *forces, nnp_stream_t stream);

/* Test hook: out[M,N] = A[M,K] * W[N,K]^T (+ bias[N]) through the same tile engine the node
 * kernels use (3xTF32 tensor-core path or FP32 FFMA). */
int nnp_test_gemm_nt(const float *A, const nnp_gemm_weight *W, const float *bias, float *out,
                     int32_t M, int32_t N, int32_t K, nnp_stream_t stream);
/* Test hook: 5 = streaming tcgen05 3xTF32 kernel for the 128 x 128 channel mixes, other shapes as 3
 * (default), 3 = tcgen05 3xTF32 with one tile per CTA, 1 = mma.sync 3xTF32, 0 = FP32 FFMA. */
int nnp_set_gemm_mode(int use_mma);

/* Instrumentation (bench.py / tests): number of kernels this library has enqueued so far
 * (reset != 0 clears it), and per-kernel device times measured with CUDA events on the
 * launching stream: nnp_profile_begin() arms it, nnp_profile_report() synchronises and writes
 * "label total_ms launches\n" lines. */
int nnp_launch_count(int reset);
int nnp_profile_begin(void);
int nnp_profile_report(char *buf, int buf_bytes);

#ifdef __cplusplus
}
#endif
#endif /* NNP_B200_H */
