"""CPU oracle for the TensorNet energy-and-forces step (float64).

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / reference arm
may import this module.

PARITY UNPINNED.  The reference package contains no TensorNet
(``/root/reference/SPEC.md:17,357`` put it out of scope; ``PAPER.md:50-54``
describes it in prose only) and upstream ``torchmdnet`` is not installed and
not vendored, so there is no golden vector to pin these numerics to.  The
equations below are the frozen specification of the path (SURVEY.md Appendix A,
restating the public ``torchmdnet/models/tensornet.py``), with the reference
package's conventions wherever the two differ:

* receivers = ``pairs[:, 0]``, senders = ``pairs[:, 1]``  (graphnet.py:353-355)
* delta = r_i - r_j, full directed list with self loops     (neighbors.py:64, 213-219)
* cosine cutoff / expnorm basis exactly as radial.py:11-73
* SiLU as _ops.py:31-37, head Linear(C->C/2)-SiLU-Linear(C/2->1), per-atom
  ``raw*std + mean`` then per-sample sum                     (graphnet.py:171, 403-411)
* sentinel edge slots are skipped                            (graphnet.py:225-267 equivalently)

What substitutes for a golden vector (tests/test_oracle_tensornet.py): two
independent implementations in this file -- ``energy_forces_torch`` (dense
3x3 tensors, forces by autograd) and ``energy_forces_compact`` (1+3+5
irreducible components, hand-derived reverse sweep; the blueprint of the CUDA
kernels) -- must agree to 1e-10; forces must match central differences; energy
must be O(3)/translation/permutation invariant; padding must be inert.

Notation: edge e = (i <- j); d_e, u_e = delta_e/d_e (0 on loops);
phi_e = cosine_cutoff(d_e); rho_e = rbf_expnorm(d_e); X_i in R^{C x 3 x 3}.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Optional

import numpy as np

from .neighbors_oracle import (
    cosine_cutoff,
    cosine_cutoff_grad,
    expnorm_initial_params,
    rbf_expnorm,
    rbf_expnorm_dd,
    segment_sum,
    silu,
    silu_grad,
)

LN_EPS = 1e-5


@dataclass(frozen=True)
class OracleConfig:
    embedding_dimension: int = 128
    num_layers: int = 2
    num_rbf: int = 32
    cutoff_lower: float = 0.0
    cutoff_upper: float = 5.0
    max_z: int = 100
    mean: float = 0.0
    std: float = 1.0


def init_params(cfg: OracleConfig, seed: int = 0) -> Dict[str, np.ndarray]:
    """Deterministic random weights in the style of graphnet.py:175-222:
    ``default_rng(seed)``, linears U(+-1/sqrt(fan_in)), embedding N(0,1),
    LayerNorm gamma=1 beta=0.  Draw order is the key order below."""
    rng = np.random.default_rng(seed)
    C, K, L = cfg.embedding_dimension, cfg.num_rbf, cfg.num_layers
    H = max(C // 2, 1)

    def lin(out_f, in_f, bias=True):
        b = 1.0 / np.sqrt(in_f)
        w = rng.uniform(-b, b, (out_f, in_f))
        return (w, rng.uniform(-b, b, out_f)) if bias else w

    p: Dict[str, np.ndarray] = {}
    p["emb"] = rng.standard_normal((cfg.max_z, C))
    p["emb2_w"], p["emb2_b"] = lin(C, 2 * C)
    dp = [lin(C, K) for _ in range(3)]
    p["dp_w"] = np.stack([w for w, _ in dp])
    p["dp_b"] = np.stack([b for _, b in dp])
    p["init_norm_g"], p["init_norm_b"] = np.ones(C), np.zeros(C)
    p["es0_w"], p["es0_b"] = lin(2 * C, C)
    p["es1_w"], p["es1_b"] = lin(3 * C, 2 * C)
    p["et_w"] = np.stack([lin(C, C, bias=False) for _ in range(3)])
    for l in range(L):
        p[f"l{l}_s0_w"], p[f"l{l}_s0_b"] = lin(C, K)
        p[f"l{l}_s1_w"], p[f"l{l}_s1_b"] = lin(2 * C, C)
        p[f"l{l}_s2_w"], p[f"l{l}_s2_b"] = lin(3 * C, 2 * C)
        p[f"l{l}_t_w"] = np.stack([lin(C, C, bias=False) for _ in range(6)])
    p["out_norm_g"], p["out_norm_b"] = np.ones(3 * C), np.zeros(3 * C)
    p["lin_w"], p["lin_b"] = lin(C, 3 * C)
    p["h1_w"], p["h1_b"] = lin(H, C)
    b = 1.0 / np.sqrt(H)
    p["h2_w"] = rng.uniform(-b, b, H)
    p["h2_b"] = np.array(rng.uniform(-b, b))
    p["rbf_means"], p["rbf_betas"] = expnorm_initial_params(K, cfg.cutoff_lower, cfg.cutoff_upper)
    return p


# =========================================================================== torch
# Literal dense form, forces by autograd.  Independent of the compact code below.

def energy_forces_torch(params, cfg: OracleConfig, species, batch, positions, pairs, deltas,
                        n_samples: Optional[int] = None, want_forces: bool = True,
                        num_threads: Optional[int] = None):
    """pairs [E,2] (valid rows only, loops included as i==j), deltas [E,3] = minimum-image
    r_i - r_j.  Returns (energy [n_samples], forces [N,3] or None, per_atom [N])."""
    import torch

    if num_threads:
        torch.set_num_threads(num_threads)
    dt = torch.float64
    P = {k: torch.as_tensor(np.asarray(v), dtype=dt) for k, v in params.items()}
    C, K, L = cfg.embedding_dimension, cfg.num_rbf, cfg.num_layers
    z = torch.as_tensor(np.asarray(species), dtype=torch.long)
    b = torch.as_tensor(np.asarray(batch), dtype=torch.long)
    pos = torch.tensor(np.asarray(positions, dtype=np.float64), dtype=dt, requires_grad=want_forces)
    pr = torch.as_tensor(np.asarray(pairs), dtype=torch.long)
    recv, send = pr[:, 0], pr[:, 1]
    N = pos.shape[0]
    n_samples = int(b.max()) + 1 if n_samples is None else n_samples
    dl = torch.as_tensor(np.asarray(deltas, dtype=np.float64), dtype=dt)
    # constant lattice shift so that delta is a differentiable function of positions
    shift = dl - (pos.detach()[recv] - pos.detach()[send])
    delta = pos[recv] - pos[send] + shift
    loop = recv == send
    safe = torch.where(loop[:, None], torch.ones_like(delta), delta)
    d = torch.where(loop, torch.zeros(len(pr), dtype=dt), safe.norm(dim=1))
    u = torch.where(loop[:, None], torch.zeros_like(delta), safe / safe.norm(dim=1, keepdim=True))

    rl, ru = cfg.cutoff_lower, cfg.cutoff_upper
    if rl == 0.0:
        phi = torch.where(d <= ru, 0.5 * (torch.cos(np.pi * d / ru) + 1.0), torch.zeros_like(d))
    else:
        t = 2.0 * (d - rl) / (ru - rl) + 1.0
        phi = torch.where((d >= rl) & (d <= ru), 0.5 * (torch.cos(np.pi * t) + 1.0), torch.zeros_like(d))
    rho = torch.exp(-P["rbf_betas"] * (torch.exp(rl - d)[:, None] - P["rbf_means"]) ** 2)

    eye = torch.eye(3, dtype=dt)

    def skew(v):
        o = torch.zeros(v.shape[0], 3, 3, dtype=dt)
        o[:, 0, 1], o[:, 0, 2] = -v[:, 2], v[:, 1]
        o[:, 1, 0], o[:, 1, 2] = v[:, 2], -v[:, 0]
        o[:, 2, 0], o[:, 2, 1] = -v[:, 1], v[:, 0]
        return o

    def decompose(M):
        tr = M.diagonal(dim1=-2, dim2=-1).sum(-1)
        I = (tr / 3.0)[..., None, None] * eye
        A = 0.5 * (M - M.transpose(-1, -2))
        S = 0.5 * (M + M.transpose(-1, -2)) - I
        return I, A, S

    def tnorm(M):
        return (M * M).sum((-1, -2))

    def mix(W, M):  # M [N,C,3,3], W [C_out, C_in]
        return torch.einsum("oc,ncab->noab", W, M)

    def layer_norm(x, g, bb):
        mu = x.mean(-1, keepdim=True)
        var = ((x - mu) ** 2).mean(-1, keepdim=True)
        return (x - mu) / torch.sqrt(var + LN_EPS) * g + bb

    act = torch.nn.functional.silu

    # ---- embedding
    Z = torch.cat([P["emb"][z[recv]], P["emb"][z[send]]], dim=1) @ P["emb2_w"].T + P["emb2_b"]
    c = phi[:, None] * Z
    w = [(rho @ P["dp_w"][k].T + P["dp_b"][k]) * c for k in range(3)]
    sym = u[:, :, None] * u[:, None, :] - (u * u).sum(1)[:, None, None] / 3.0 * eye
    Ie = w[0][:, :, None, None] * eye
    Ae = w[1][:, :, None, None] * skew(u)[:, None]
    Se = w[2][:, :, None, None] * sym[:, None]
    zero = torch.zeros(N, C, 3, 3, dtype=dt)
    I = zero.index_add(0, recv, Ie)
    A = zero.index_add(0, recv, Ae)
    S = zero.index_add(0, recv, Se)
    nrm = layer_norm(tnorm(I + A + S), P["init_norm_g"], P["init_norm_b"])
    nrm = act(act(nrm @ P["es0_w"].T + P["es0_b"]) @ P["es1_w"].T + P["es1_b"]).reshape(N, C, 3)
    X = (mix(P["et_w"][0], I) * nrm[:, :, 0, None, None]
         + mix(P["et_w"][1], A) * nrm[:, :, 1, None, None]
         + mix(P["et_w"][2], S) * nrm[:, :, 2, None, None])

    # ---- interaction layers
    for l in range(L):
        f = act(act(act(rho @ P[f"l{l}_s0_w"].T + P[f"l{l}_s0_b"]) @ P[f"l{l}_s1_w"].T
                    + P[f"l{l}_s1_b"]) @ P[f"l{l}_s2_w"].T + P[f"l{l}_s2_b"])
        f = (f * phi[:, None]).reshape(-1, C, 3)
        Xh = X / (tnorm(X) + 1.0)[..., None, None]
        I, A, S = decompose(Xh)
        T = P[f"l{l}_t_w"]
        I, A, S = mix(T[0], I), mix(T[1], A), mix(T[2], S)
        Y = I + A + S
        msg = (f[:, :, 0, None, None] * I[send] + f[:, :, 1, None, None] * A[send]
               + f[:, :, 2, None, None] * S[send])
        M = zero.index_add(0, recv, msg)
        Pm = M @ Y + Y @ M
        I, A, S = decompose(Pm)
        nn_ = (tnorm(I + A + S) + 1.0)[..., None, None]
        dX = mix(T[3], I / nn_) + mix(T[4], A / nn_) + mix(T[5], S / nn_)
        X = Xh + dX + dX @ dX

    # ---- readout
    I, A, S = decompose(X)
    x = torch.cat([tnorm(I), tnorm(A), tnorm(S)], dim=-1)
    x = layer_norm(x, P["out_norm_g"], P["out_norm_b"])
    x = act(x @ P["lin_w"].T + P["lin_b"])
    raw = act(x @ P["h1_w"].T + P["h1_b"]) @ P["h2_w"] + P["h2_b"]
    per_atom = raw * cfg.std + cfg.mean
    energy = torch.zeros(n_samples, dtype=dt).index_add(0, b, per_atom)
    forces = None
    if want_forces:
        (grad,) = torch.autograd.grad(energy.sum(), pos)
        forces = (-grad).numpy()
    return energy.detach().numpy(), forces, per_atom.detach().numpy()


# ========================================================================= compact
# Irreducible components per channel, c9 = [s | ax ay az | Sxx Syy Sxy Sxz Syz]:
#   M = s*1 + skew(a) + S,  skew(a) = [[0,-az,ay],[az,0,-ax],[-ay,ax,0]],  Szz = -Sxx-Syy.
# Gradients are stored the same way: the components of the Frobenius gradient MATRIX
# G = dL/dM.  Channel mixing acts on each component alike, so its transpose does too,
# and the three subspaces are Frobenius-orthogonal, so projections commute with it.

def to_full(c9):
    """[..., 9] -> [..., 3, 3]."""
    s, ax, ay, az, sxx, syy, sxy, sxz, syz = np.moveaxis(c9, -1, 0)
    szz = -sxx - syy
    M = np.empty(c9.shape[:-1] + (3, 3))
    M[..., 0, 0] = s + sxx
    M[..., 1, 1] = s + syy
    M[..., 2, 2] = s + szz
    M[..., 0, 1] = sxy - az
    M[..., 1, 0] = sxy + az
    M[..., 0, 2] = sxz + ay
    M[..., 2, 0] = sxz - ay
    M[..., 1, 2] = syz - ax
    M[..., 2, 1] = syz + ax
    return M


def from_full(M):
    """[..., 3, 3] -> [..., 9] (exact inverse of to_full)."""
    s = (M[..., 0, 0] + M[..., 1, 1] + M[..., 2, 2]) / 3.0
    out = np.empty(M.shape[:-2] + (9,))
    out[..., 0] = s
    out[..., 1] = 0.5 * (M[..., 2, 1] - M[..., 1, 2])
    out[..., 2] = 0.5 * (M[..., 0, 2] - M[..., 2, 0])
    out[..., 3] = 0.5 * (M[..., 1, 0] - M[..., 0, 1])
    out[..., 4] = M[..., 0, 0] - s
    out[..., 5] = M[..., 1, 1] - s
    out[..., 6] = 0.5 * (M[..., 0, 1] + M[..., 1, 0])
    out[..., 7] = 0.5 * (M[..., 0, 2] + M[..., 2, 0])
    out[..., 8] = 0.5 * (M[..., 1, 2] + M[..., 2, 1])
    return out


def dot_I(a, b):
    return 3.0 * a[..., 0] * b[..., 0]


def dot_A(a, b):
    return 2.0 * (a[..., 1] * b[..., 1] + a[..., 2] * b[..., 2] + a[..., 3] * b[..., 3])


def dot_S(a, b):
    azz, bzz = a[..., 4] + a[..., 5], b[..., 4] + b[..., 5]
    return (a[..., 4] * b[..., 4] + a[..., 5] * b[..., 5] + azz * bzz
            + 2.0 * (a[..., 6] * b[..., 6] + a[..., 7] * b[..., 7] + a[..., 8] * b[..., 8]))


def frob(a, b):
    return dot_I(a, b) + dot_A(a, b) + dot_S(a, b)


GROUP = np.array([0, 1, 1, 1, 2, 2, 2, 2, 2])   # component -> I/A/S


def mix3(T, x9):
    """x9 [N,C,9]; T [3,C,C]: component q is mixed with T[GROUP[q]]."""
    out = np.empty_like(x9)
    for q in range(9):
        out[:, :, q] = x9[:, :, q] @ T[GROUP[q]].T
    return out


def mix3_T(T, g9):
    out = np.empty_like(g9)
    for q in range(9):
        out[:, :, q] = g9[:, :, q] @ T[GROUP[q]]
    return out


def edge_basis(u, loop):
    """Per-edge 9-vector of the unit tensors: [1 | u | sym5(u)] (zero A,S parts on loops)."""
    E = u.shape[0]
    b = np.zeros((E, 9))
    b[:, 0] = 1.0
    b[:, 1:4] = u
    uu = (u * u).sum(1)
    b[:, 4] = u[:, 0] ** 2 - uu / 3.0
    b[:, 5] = u[:, 1] ** 2 - uu / 3.0
    b[:, 6] = u[:, 0] * u[:, 1]
    b[:, 7] = u[:, 0] * u[:, 2]
    b[:, 8] = u[:, 1] * u[:, 2]
    b[loop, 1:] = 0.0
    return b


def _ln_fwd(x, g, b):
    mu = x.mean(-1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xh = xc * rstd
    return xh * g + b, (xh, rstd)


def _ln_bwd(gy, g, cache):
    xh, rstd = cache
    gxh = gy * g
    return rstd * (gxh - gxh.mean(-1, keepdims=True) - xh * (gxh * xh).mean(-1, keepdims=True))


def radial_mlp(params, l, rho):
    """f~(rho) before the envelope: SiLU(ls2(SiLU(ls1(SiLU(ls0(rho))))))  [E,3C]."""
    a0 = rho @ params[f"l{l}_s0_w"].T + params[f"l{l}_s0_b"]
    a1 = silu(a0) @ params[f"l{l}_s1_w"].T + params[f"l{l}_s1_b"]
    a2 = silu(a1) @ params[f"l{l}_s2_w"].T + params[f"l{l}_s2_b"]
    return silu(a2), (a0, a1, a2)


def radial_mlp_dd(params, l, rho, drho_dd, cache):
    """d f~ / d d by forward-mode through the MLP."""
    a0, a1, a2 = cache
    t = drho_dd @ params[f"l{l}_s0_w"].T
    t = (t * silu_grad(a0)) @ params[f"l{l}_s1_w"].T
    t = (t * silu_grad(a1)) @ params[f"l{l}_s2_w"].T
    return t * silu_grad(a2)


def energy_forces_compact(params, cfg: OracleConfig, species, batch, pairs, deltas, dists,
                          n_samples: Optional[int] = None, want_forces: bool = True,
                          return_intermediates: bool = False, edge_chunk: int = 32768):
    """Same function as energy_forces_torch in irreducible components, with the reverse
    sweep written out by hand.  ``dists`` must equal |deltas| (0 on loops).  Edge-level
    temporaries are produced ``edge_chunk`` edges at a time (and the radial MLP recomputed in
    the reverse sweep) so that systems with millions of edges fit in host memory."""
    C, K, L = cfg.embedding_dimension, cfg.num_rbf, cfg.num_layers
    P = params
    z = np.asarray(species, dtype=np.int64)
    b = np.asarray(batch, dtype=np.int64)
    pr = np.asarray(pairs, dtype=np.int64)
    recv, send = pr[:, 0], pr[:, 1]
    N = z.shape[0]
    E = pr.shape[0]
    n_samples = int(b.max()) + 1 if n_samples is None else n_samples
    dl = np.asarray(deltas, dtype=np.float64)
    d = np.asarray(dists, dtype=np.float64)
    loop = recv == send
    safe = np.where(loop, 1.0, d)
    u = dl / safe[:, None]
    u[loop] = 0.0
    rl, ru = cfg.cutoff_lower, cfg.cutoff_upper
    phi = cosine_cutoff(d, rl, ru)
    dphi = cosine_cutoff_grad(d, rl, ru)
    basis = edge_basis(u, loop)                                   # [E,9]
    chunks = [slice(s, min(s + edge_chunk, E)) for s in range(0, E, edge_chunk)]
    gI = GROUP == 0
    gA = GROUP == 1
    gS = GROUP == 2

    def rho_of(sl):
        return (rbf_expnorm(d[sl], P["rbf_means"], P["rbf_betas"], rl),
                rbf_expnorm_dd(d[sl], P["rbf_means"], P["rbf_betas"], rl))

    # ------------------------------------------------------------------ forward
    Wa, Wb = P["emb2_w"][:, :C], P["emb2_w"][:, C:]
    Zt_r = P["emb"] @ Wa.T                                         # hoisted tables [max_z, C]
    Zt_s = P["emb"] @ Wb.T

    def embed_weights(sl):
        rho, drho = rho_of(sl)
        Z = Zt_r[z[recv[sl]]] + Zt_s[z[send[sl]]] + P["emb2_b"]              # [e,C]
        dpv = np.stack([rho @ P["dp_w"][k].T + P["dp_b"][k] for k in range(3)], axis=-1)
        ddp = np.stack([drho @ P["dp_w"][k].T for k in range(3)], axis=-1)
        return Z, dpv, ddp

    X0 = np.zeros((N, C * 9))
    for sl in chunks:
        Z, dpv, _ = embed_weights(sl)
        w = dpv * (phi[sl, None] * Z)[:, :, None]                            # [e,C,3]
        contrib = w[:, :, GROUP] * basis[sl, None, :]
        X0 += segment_sum(contrib.reshape(-1, C * 9), recv[sl], N)
    X0 = X0.reshape(N, C, 9)
    n0 = frob(X0, X0)                                              # [N,C]
    ln0, ln0_cache = _ln_fwd(n0, P["init_norm_g"], P["init_norm_b"])
    e0 = ln0 @ P["es0_w"].T + P["es0_b"]
    e1 = silu(e0) @ P["es1_w"].T + P["es1_b"]
    gate = silu(e1).reshape(N, C, 3)
    Xm = mix3(P["et_w"], X0)
    X = Xm * gate[:, :, GROUP]

    saved = []
    for l in range(L):
        nx = frob(X, X) + 1.0
        Xh = X / nx[:, :, None]
        T = P[f"l{l}_t_w"]
        Yc = mix3(T[:3], Xh)                                       # I',A',S' components
        Mc = np.zeros((N, C * 9))
        for sl in chunks:
            ft, _ = radial_mlp(P, l, rho_of(sl)[0])
            f = (ft * phi[sl, None]).reshape(-1, C, 3)
            msg = f[:, :, GROUP] * Yc[send[sl]]
            Mc += segment_sum(msg.reshape(-1, C * 9), recv[sl], N)
        Mc = Mc.reshape(N, C, 9)
        Mf, Yf = to_full(Mc), to_full(Yc)
        Pf = Mf @ Yf + Yf @ Mf
        Pc = from_full(Pf)
        npn = frob(Pc, Pc) + 1.0
        Qc = Pc / npn[:, :, None]
        Dc = mix3(T[3:], Qc)
        Df = to_full(Dc)
        Xn = Xh + Dc + from_full(Df @ Df)
        saved.append(dict(X=X, nx=nx, Xh=Xh, Yc=Yc, Mc=Mc, Pc=Pc, npn=npn, Dc=Dc))
        X = Xn

    XI, XA, XS = X * gI, X * gA, X * gS
    feats = np.concatenate([dot_I(XI, XI), dot_A(XA, XA), dot_S(XS, XS)], axis=-1)  # [N,3C]
    lnr, lnr_cache = _ln_fwd(feats, P["out_norm_g"], P["out_norm_b"])
    r0 = lnr @ P["lin_w"].T + P["lin_b"]
    r1 = silu(r0) @ P["h1_w"].T + P["h1_b"]
    raw = silu(r1) @ P["h2_w"] + P["h2_b"]
    per_atom = raw * cfg.std + cfg.mean
    energy = segment_sum(per_atom, b, n_samples)
    if not want_forces:
        return (energy, None, per_atom) if not return_intermediates else (energy, None, per_atom, {})

    # ------------------------------------------------------------------ reverse
    g_raw = np.full(N, cfg.std)
    g_r1 = (g_raw[:, None] * P["h2_w"][None, :]) * silu_grad(r1)
    g_r0 = (g_r1 @ P["h1_w"]) * silu_grad(r0)
    g_feats = _ln_bwd(g_r0 @ P["lin_w"], P["out_norm_g"], lnr_cache)          # [N,3C]
    # d(||part||^2)/dX as a Frobenius-gradient matrix: 2 * weight * part
    GX = 2.0 * (g_feats[:, :C, None] * XI + g_feats[:, C:2 * C, None] * XA
                + g_feats[:, 2 * C:, None] * XS)

    g_d = np.zeros(E)          # dE/dd_e   (directed edge, own term)
    g_u = np.zeros((E, 3))     # dE/du_e

    for l in range(L - 1, -1, -1):
        sv = saved[l]
        T = P[f"l{l}_t_w"]
        Df = to_full(sv["Dc"])
        Gf = to_full(GX)
        G_Xh = GX.copy()
        G_D = GX + from_full(Gf @ np.swapaxes(Df, -1, -2) + np.swapaxes(Df, -1, -2) @ Gf)
        G_Q = mix3_T(T[3:], G_D)
        npn, Pc = sv["npn"], sv["Pc"]
        G_P = G_Q / npn[:, :, None] - Pc * (2.0 * frob(G_Q, Pc) / npn**2)[:, :, None]
        GPf = to_full(G_P)
        Mf, Yf = to_full(sv["Mc"]), to_full(sv["Yc"])
        G_M = from_full(GPf @ np.swapaxes(Yf, -1, -2) + np.swapaxes(Yf, -1, -2) @ GPf)
        G_Y = from_full(np.swapaxes(Mf, -1, -2) @ GPf + GPf @ np.swapaxes(Mf, -1, -2))
        # edge op  M_i = sum_e f_e[:,grp] * Yc_j
        G_Y = G_Y.reshape(N, C * 9)
        for sl in chunks:
            rho, drho = rho_of(sl)
            ft, mlp_cache = radial_mlp(P, l, rho)
            f = (ft * phi[sl, None]).reshape(-1, C, 3)
            GMr, Ys = G_M[recv[sl]], sv["Yc"][send[sl]]
            G_Y += segment_sum((f[:, :, GROUP] * GMr).reshape(-1, C * 9), send[sl], N)
            g_f = np.stack([dot_I(GMr, Ys), dot_A(GMr, Ys), dot_S(GMr, Ys)], axis=-1)   # [e,C,3]
            dft = radial_mlp_dd(P, l, rho, drho, mlp_cache).reshape(-1, C, 3)
            ft3 = ft.reshape(-1, C, 3)
            g_d[sl] += (g_f * (dft * phi[sl, None, None] + ft3 * dphi[sl, None, None])).sum((1, 2))
        G_Y = G_Y.reshape(N, C, 9)
        G_Xh += mix3_T(T[:3], G_Y)
        nx, Xin = sv["nx"], sv["X"]
        GX = G_Xh / nx[:, :, None] - Xin * (2.0 * frob(G_Xh, Xin) / nx**2)[:, :, None]

    # embedding:  X = mix3(et, X0) * gate[grp]
    G_Xm = GX * gate[:, :, GROUP]
    g_gate = np.stack([dot_I(GX, Xm), dot_A(GX, Xm), dot_S(GX, Xm)], axis=-1)       # [N,C,3]
    g_e1 = g_gate.reshape(N, 3 * C) * silu_grad(e1)
    g_e0 = (g_e1 @ P["es1_w"]) * silu_grad(e0)
    g_n0 = _ln_bwd(g_e0 @ P["es0_w"], P["init_norm_g"], ln0_cache)                   # [N,C]
    G_X0 = mix3_T(P["et_w"], G_Xm) + 2.0 * g_n0[:, :, None] * X0
    # edge accumulation X0_i += w_e[:,grp] * basis_e
    for sl in chunks:
        Z, dpv, ddp = embed_weights(sl)
        w = dpv * (phi[sl, None] * Z)[:, :, None]
        Gr = G_X0[recv[sl]]                                                          # [e,C,9]
        bs = basis[sl]
        bI = np.zeros_like(bs)
        bI[:, 0] = 1.0
        g_w = np.stack([dot_I(Gr, bI[:, None, :]), dot_A(Gr, (bs * gA)[:, None, :]),
                        dot_S(Gr, (bs * gS)[:, None, :])], axis=-1)                  # [e,C,3]
        g_d[sl] += (g_w * Z[:, :, None] * (ddp * phi[sl, None, None] + dpv * dphi[sl, None, None])).sum((1, 2))
        # d/du of  2*w2*(a_G . u)  and  w3 * u^T S_G u
        g_u[sl] += 2.0 * np.einsum("ec,ecq->eq", w[:, :, 1], Gr[:, :, 1:4])
        SG = to_full(Gr * gS)                                                        # [e,C,3,3]
        g_u[sl] += 2.0 * np.einsum("ec,ecab,eb->ea", w[:, :, 2], SG, u[sl])
    g_u[loop] = 0.0

    # pullback: d = |delta|, u = delta/d
    proj = g_u - u * (g_u * u).sum(1)[:, None]
    p = g_d[:, None] * u + proj / safe[:, None]
    p[loop] = 0.0
    grad = segment_sum(p, recv, N) - segment_sum(p, send, N)
    forces = -grad
    if return_intermediates:
        return energy, forces, per_atom, dict(g_d=g_d, g_u=g_u, X0=X0, X=X, saved=saved)
    return energy, forces, per_atom
