// Per-channel 3x3 tensor algebra of TensorNet in irreducible components.
//
// A 3x3 matrix M (one per node and channel) is stored as nine numbers
//   c9 = [ s | ax ay az | Sxx Syy Sxy Sxz Syz ],   M = s*1 + skew(a) + S,
//   skew(a) = [[0,-az,ay],[az,0,-ax],[-ay,ax,0]],  Szz = -Sxx-Syy
// i.e. the I / A / S decomposition of SURVEY.md Appendix A (1 + 3 + 5 components) is the
// storage format itself.  Gradients use the same format: the components of the Frobenius
// gradient matrix dL/dM.  Channel mixing acts on every component alike and the three
// subspaces are Frobenius-orthogonal, so forward and reverse sweeps never leave this basis.
//
// Everything here is plain inline arithmetic usable from host code as well, so the formulas
// can be unit-tested on a CPU-only box against the oracle (tests/test_tn_math_host.py).
#pragma once

#include <math.h>

#if defined(__CUDACC__)
#define NNP_HD __host__ __device__ __forceinline__
#else
#define NNP_HD inline
#endif

struct Mat3 {
    float m[3][3];
};

NNP_HD void c9_to_full(const float *c, Mat3 &M)
{
    const float s = c[0], ax = c[1], ay = c[2], az = c[3];
    const float sxx = c[4], syy = c[5], sxy = c[6], sxz = c[7], syz = c[8];
    M.m[0][0] = s + sxx;
    M.m[1][1] = s + syy;
    M.m[2][2] = s - sxx - syy;
    M.m[0][1] = sxy - az;
    M.m[1][0] = sxy + az;
    M.m[0][2] = sxz + ay;
    M.m[2][0] = sxz - ay;
    M.m[1][2] = syz - ax;
    M.m[2][1] = syz + ax;
}

NNP_HD void full_to_c9(const Mat3 &M, float *c)
{
    const float s = (M.m[0][0] + M.m[1][1] + M.m[2][2]) * (1.0f / 3.0f);
    c[0] = s;
    c[1] = 0.5f * (M.m[2][1] - M.m[1][2]);
    c[2] = 0.5f * (M.m[0][2] - M.m[2][0]);
    c[3] = 0.5f * (M.m[1][0] - M.m[0][1]);
    c[4] = M.m[0][0] - s;
    c[5] = M.m[1][1] - s;
    c[6] = 0.5f * (M.m[0][1] + M.m[1][0]);
    c[7] = 0.5f * (M.m[0][2] + M.m[2][0]);
    c[8] = 0.5f * (M.m[1][2] + M.m[2][1]);
}

// Frobenius inner products restricted to the I, A and S parts.
NNP_HD float c9_dot_I(const float *a, const float *b) { return 3.0f * a[0] * b[0]; }
NNP_HD float c9_dot_A(const float *a, const float *b)
{
    return 2.0f * (a[1] * b[1] + a[2] * b[2] + a[3] * b[3]);
}
NNP_HD float c9_dot_S(const float *a, const float *b)
{
    const float azz = a[4] + a[5], bzz = b[4] + b[5];
    return a[4] * b[4] + a[5] * b[5] + azz * bzz +
           2.0f * (a[6] * b[6] + a[7] * b[7] + a[8] * b[8]);
}
NNP_HD float c9_frob(const float *a, const float *b)
{
    return c9_dot_I(a, b) + c9_dot_A(a, b) + c9_dot_S(a, b);
}

NNP_HD void mat3_mul(const Mat3 &A, const Mat3 &B, Mat3 &C)
{
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int i = 0; i < 3; ++i) {
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
        for (int j = 0; j < 3; ++j)
            C.m[i][j] = A.m[i][0] * B.m[0][j] + A.m[i][1] * B.m[1][j] + A.m[i][2] * B.m[2][j];
    }
}

// C = A*B + B*A
NNP_HD void mat3_anticomm(const Mat3 &A, const Mat3 &B, Mat3 &C)
{
    Mat3 ab, ba;
    mat3_mul(A, B, ab);
    mat3_mul(B, A, ba);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) C.m[i][j] = ab.m[i][j] + ba.m[i][j];
}

// C = G*B^T + B^T*G   (reverse of P = A*B + B*A with respect to A, and with A<->B for B)
NNP_HD void mat3_anticomm_T(const Mat3 &G, const Mat3 &B, Mat3 &C)
{
    Mat3 bt;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) bt.m[i][j] = B.m[j][i];
    mat3_anticomm(G, bt, C);
}

// Unit tensors of an edge with unit vector u: [1 | u | sym5(u)]  (all zero but b[0] on loops).
NNP_HD void edge_basis9(float ux, float uy, float uz, float *b)
{
    const float uu = (ux * ux + uy * uy + uz * uz) * (1.0f / 3.0f);
    b[0] = 1.0f;
    b[1] = ux;
    b[2] = uy;
    b[3] = uz;
    b[4] = ux * ux - uu;
    b[5] = uy * uy - uu;
    b[6] = ux * uy;
    b[7] = ux * uz;
    b[8] = uy * uz;
}

NNP_HD float nnp_sigmoid(float x)
{
    return 1.0f / (1.0f + expf(-x));
}
NNP_HD float nnp_silu(float x) { return x * nnp_sigmoid(x); }
NNP_HD float nnp_silu_grad(float x)
{
    const float s = nnp_sigmoid(x);
    return s * (1.0f + x * (1.0f - s));
}

// Cubic Hermite basis on t in [0,1]; m0/m1 are slopes pre-multiplied by the knot spacing.
struct Hermite {
    float h00, h10, h01, h11;   // value weights for f0, m0, f1, m1
    float d00, d10, d01, d11;   // d/dt weights
};

NNP_HD Hermite hermite_weights(float t)
{
    Hermite h;
    const float t2 = t * t, t3 = t2 * t;
    h.h00 = 2.0f * t3 - 3.0f * t2 + 1.0f;
    h.h10 = t3 - 2.0f * t2 + t;
    h.h01 = -2.0f * t3 + 3.0f * t2;
    h.h11 = t3 - t2;
    h.d00 = 6.0f * t2 - 6.0f * t;
    h.d10 = 3.0f * t2 - 4.0f * t + 1.0f;
    h.d01 = -h.d00;
    h.d11 = 3.0f * t2 - 2.0f * t;
    return h;
}

// Forward of one interaction layer's node update, per (node, channel):
//   P = M*Y + Y*M ; Q = P / (|P|^2 + 1)
NNP_HD void node_product_fwd(const float *Mc, const float *Yc, float *Qc)
{
    Mat3 M, Y, P;
    c9_to_full(Mc, M);
    c9_to_full(Yc, Y);
    mat3_anticomm(M, Y, P);
    float Pc[9];
    full_to_c9(P, Pc);
    const float inv = 1.0f / (c9_frob(Pc, Pc) + 1.0f);
    for (int q = 0; q < 9; ++q) Qc[q] = Pc[q] * inv;
}

// Reverse: given G_Q, recompute P and return G_M and G_Y (the part of dL/dY through P).
NNP_HD void node_product_bwd(const float *Mc, const float *Yc, const float *GQ, float *GM, float *GY)
{
    Mat3 M, Y, P, GP, T;
    c9_to_full(Mc, M);
    c9_to_full(Yc, Y);
    mat3_anticomm(M, Y, P);
    float Pc[9], GPc[9];
    full_to_c9(P, Pc);
    const float n = c9_frob(Pc, Pc) + 1.0f;
    const float inv = 1.0f / n;
    const float k = 2.0f * c9_frob(GQ, Pc) * inv * inv;
    for (int q = 0; q < 9; ++q) GPc[q] = GQ[q] * inv - Pc[q] * k;
    c9_to_full(GPc, GP);
    mat3_anticomm_T(GP, Y, T);   // G_M = GP*Y^T + Y^T*GP
    full_to_c9(T, GM);
    mat3_anticomm_T(GP, M, T);   // G_Y = GP*M^T + M^T*GP
    full_to_c9(T, GY);
}

// X_new = Xh + D + D*D
NNP_HD void residual_fwd(const float *Xh, const float *Dc, float *Xn)
{
    Mat3 D, DD;
    c9_to_full(Dc, D);
    mat3_mul(D, D, DD);
    float t[9];
    full_to_c9(DD, t);
    for (int q = 0; q < 9; ++q) Xn[q] = Xh[q] + Dc[q] + t[q];
}

// G_D = G + G*D^T + D^T*G   (G is dL/dX_new; dL/dXh = G itself)
NNP_HD void residual_bwd(const float *G, const float *Dc, float *GD)
{
    Mat3 Gf, D, T;
    c9_to_full(G, Gf);
    c9_to_full(Dc, D);
    mat3_anticomm_T(Gf, D, T);
    float t[9];
    full_to_c9(T, t);
    for (int q = 0; q < 9; ++q) GD[q] = G[q] + t[q];
}

// Xh = X / (|X|^2 + 1)
NNP_HD float normalize_fwd(const float *X, float *Xh)
{
    const float n = c9_frob(X, X) + 1.0f;
    const float inv = 1.0f / n;
    for (int q = 0; q < 9; ++q) Xh[q] = X[q] * inv;
    return n;
}

// dL/dX from dL/dXh, with X = Xh*n
NNP_HD void normalize_bwd(const float *GXh, const float *Xh, float n, float *GX)
{
    // X = Xh*n  =>  (2<G,X>/n^2) X = 2<G,Xh> Xh
    const float inv = 1.0f / n;
    const float k = 2.0f * c9_frob(GXh, Xh);
    for (int q = 0; q < 9; ++q) GX[q] = GXh[q] * inv - Xh[q] * k;
}
