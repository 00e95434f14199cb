// Host build of csrc/tn_math.cuh so the per-channel tensor algebra can be checked against the
// CPU oracle without a GPU.  Test infrastructure only.
#include "../../paper_2402_17660_b200/csrc/tn_math.cuh"

extern "C" {
void h_to_full(const float *c, float *m) { Mat3 M; c9_to_full(c, M); for (int i = 0; i < 9; ++i) m[i] = M.m[i / 3][i % 3]; }
void h_from_full(const float *m, float *c) { Mat3 M; for (int i = 0; i < 9; ++i) M.m[i / 3][i % 3] = m[i]; full_to_c9(M, c); }
float h_frob(const float *a, const float *b) { return c9_frob(a, b); }
void h_dots(const float *a, const float *b, float *o) { o[0] = c9_dot_I(a, b); o[1] = c9_dot_A(a, b); o[2] = c9_dot_S(a, b); }
void h_basis(float x, float y, float z, float *b) { edge_basis9(x, y, z, b); }
void h_node_product_fwd(const float *M, const float *Y, float *Q) { node_product_fwd(M, Y, Q); }
void h_node_product_bwd(const float *M, const float *Y, const float *GQ, float *GM, float *GY) { node_product_bwd(M, Y, GQ, GM, GY); }
void h_residual_fwd(const float *Xh, const float *D, float *Xn) { residual_fwd(Xh, D, Xn); }
void h_residual_bwd(const float *G, const float *D, float *GD) { residual_bwd(G, D, GD); }
float h_normalize_fwd(const float *X, float *Xh) { return normalize_fwd(X, Xh); }
void h_normalize_bwd(const float *G, const float *Xh, float n, float *GX) { normalize_bwd(G, Xh, n, GX); }
void h_hermite(float t, float *w) { Hermite h = hermite_weights(t); w[0]=h.h00; w[1]=h.h10; w[2]=h.h01; w[3]=h.h11; w[4]=h.d00; w[5]=h.d10; w[6]=h.d01; w[7]=h.d11; }
float h_silu(float x) { return nnp_silu(x); }
float h_silu_grad(float x) { return nnp_silu_grad(x); }
}
