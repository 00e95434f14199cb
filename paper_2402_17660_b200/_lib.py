"""ctypes binding of ``libnnp_b200.so`` -- the C ABI declared in ``include/nnp_b200.h``.

There is no fallback: if the library is missing or a call fails, ``ExtensionError`` is raised.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ExtensionError, ValidationError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnnp_b200.so")

NNP_OK = 0
NNP_ERR_INVALID = -1
NNP_ERR_WORKSPACE = -2
NNP_ERR_CUDA = -3

BOX_KIND = {"none": 0, "orthorhombic": 1, "triclinic": 2}
STRATEGY_BRUTE, STRATEGY_CELL = 0, 1
NL_FULL_LIST, NL_SELF_LOOPS, NL_RENUMBER, NL_F32_OUT, NL_NO_PAD, NL_UNSORTED = 1, 2, 4, 8, 16, 32
TN_MAX_LAYERS = 8

EXPORTED_SYMBOLS = (
    "nnp_last_error", "nnp_version", "nnp_abi_sizeof", "nnp_nl_workspace_bytes", "nnp_nl_build", "nnp_f32_to_f64",
    "nnp_distance_pullback", "nnp_distance_pullback_second", "nnp_tn_workspace_bytes", "nnp_tn_energy_forces",
    "nnp_test_gemm_nt", "nnp_set_gemm_mode", "nnp_launch_count", "nnp_profile_begin",
    "nnp_profile_report", "nnp_md_langevin_middle", "nnp_priors_pair_terms",
)

_f = ctypes.c_float
_p = ctypes.c_void_p
_i32 = ctypes.c_int32


class NlParams(ctypes.Structure):
    _fields_ = [
        ("n_atoms", _i32), ("n_samples", _i32), ("capacity", _i32), ("box_kind", _i32),
        ("strategy", _i32), ("flags", _i32), ("grid_dims", _i32 * 3), ("max_cells", _i32),
        ("cutoff_lower", ctypes.c_double), ("cutoff_upper", ctypes.c_double),
        ("box", ctypes.c_double * 9), ("inv_box", ctypes.c_double * 9),
    ]


class PriorParams(ctypes.Structure):
    _fields_ = [("flags", ctypes.c_int32), ("reserved", ctypes.c_int32), ("cutoff_upper", ctypes.c_double),
                ("coulomb_constant", ctypes.c_double), ("switch_radius", ctypes.c_double),
                ("zbl_prefactor", ctypes.c_double), ("d2_s6", ctypes.c_double), ("d2_steep", ctypes.c_double)]


PRIOR_COULOMB, PRIOR_ZBL, PRIOR_D2 = 1, 2, 4


class GemmWeight(ctypes.Structure):
    _fields_ = [("w", _p)]


class TnModel(ctypes.Structure):
    _fields_ = [
        ("channels", _i32), ("num_rbf", _i32), ("num_layers", _i32), ("max_z", _i32),
        ("num_knots", _i32),
        ("cutoff_lower", _f), ("cutoff_upper", _f), ("u_min", _f), ("u_step", _f),
        ("mean", _f), ("std", _f), ("h2_b", _f),
        ("z_recv", _p), ("z_send", _p), ("tables", _p), ("tables_mono", _p),
        ("init_norm_g", _p), ("init_norm_b", _p),
        ("es0_w", GemmWeight), ("es0_wT", GemmWeight),
        ("es1_w", GemmWeight), ("es1_wT", GemmWeight),
        ("es0_b", _p), ("es1_b", _p),
        ("et_w", GemmWeight * 3), ("et_wT", GemmWeight * 3),
        ("layer_t_w", (GemmWeight * 6) * TN_MAX_LAYERS),
        ("layer_t_wT", (GemmWeight * 6) * TN_MAX_LAYERS),
        ("out_norm_g", _p), ("out_norm_b", _p),
        ("lin_w", GemmWeight), ("lin_wT", GemmWeight),
        ("h1_w", GemmWeight), ("h1_wT", GemmWeight),
        ("lin_b", _p), ("h1_b", _p),
        ("h2_w", _p),
        ("embed_projection", _i32), ("gemm_mode", _i32),
        ("dp_wT", _p), ("dp_b", _p), ("rbf_means", _p), ("rbf_betas", _p),
    ]


_lib = None


DEFAULT_GEMM_MODE = 5   # streaming tcgen05 kernel for the 128 x 128 mixes, per-tile tcgen05 otherwise


def load() -> ctypes.CDLL:
    """Load the extension once; fail loudly when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ExtensionError(
            f"CUDA extension not built: {LIB_PATH} is missing. Build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (needs nvcc). "
            "There is no CPU fallback."
        )
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as err:
        raise ExtensionError(f"cannot load {LIB_PATH}: {err}") from err
    sz = ctypes.c_size_t
    lib.nnp_last_error.restype = ctypes.c_char_p
    lib.nnp_last_error.argtypes = []
    lib.nnp_version.restype = ctypes.c_int
    lib.nnp_nl_workspace_bytes.argtypes = [ctypes.POINTER(NlParams), ctypes.POINTER(sz)]
    lib.nnp_nl_build.argtypes = [ctypes.POINTER(NlParams), _p, _p, _p, _p, _p, _p, _p, _p, _p, sz, _p]
    lib.nnp_f32_to_f64.argtypes = [_p, _p, ctypes.c_int64, _p]
    lib.nnp_distance_pullback.argtypes = [_p, _p, _p, _p, _i32, _i32, _p, _p, _p]
    lib.nnp_distance_pullback_second.argtypes = [_p, _p, _p, _p, _p, _i32, _i32, _i32, _p, _p, _p, _p]
    lib.nnp_tn_workspace_bytes.argtypes = [ctypes.POINTER(TnModel), _i32, _i32, _i32, ctypes.POINTER(sz)]
    lib.nnp_tn_energy_forces.argtypes = [
        ctypes.POINTER(TnModel), _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, sz, _p,
    ]
    lib.nnp_test_gemm_nt.argtypes = [_p, ctypes.POINTER(GemmWeight), _p, _p, _i32, _i32, _i32, _p]
    lib.nnp_set_gemm_mode.argtypes = [ctypes.c_int]
    dbl, u64 = ctypes.c_double, ctypes.c_uint64
    lib.nnp_priors_pair_terms.argtypes = [ctypes.POINTER(PriorParams), _p, _p, _p, _p, _i32, _i32, _p, _p, _p, _p, _p,
                                          _i32, _p, _p, _p]
    lib.nnp_md_langevin_middle.argtypes = [_p, _p, _p, _p, _p, _p, u64, _p, dbl, dbl, dbl, _p, _p, _i32, _p, _i32, _p]
    lib.nnp_launch_count.argtypes = [ctypes.c_int]
    lib.nnp_profile_begin.argtypes = []
    lib.nnp_profile_report.argtypes = [ctypes.c_char_p, ctypes.c_int]
    for name in EXPORTED_SYMBOLS:
        fn = getattr(lib, name)
        if name not in ("nnp_last_error",):
            fn.restype = ctypes.c_int
    if "NNP_GEMM_MODE" in os.environ:       # 5/3 = tcgen05, 1 = mma.sync, 0 = FFMA (measurements)
        lib.nnp_set_gemm_mode(int(os.environ["NNP_GEMM_MODE"]))
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    """Map a C return code to the package's exceptions."""
    if rc == NNP_OK:
        return
    msg = load().nnp_last_error().decode("utf-8", "replace")
    if rc == NNP_ERR_INVALID:
        raise ValidationError(f"{what}: {msg}")
    raise ExtensionError(f"{what} failed (code {rc}): {msg}")


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise ExtensionError(
            "no CUDA device available: this package runs on a B200 only (no CPU fallback)"
        )
    return torch


def ptr(t) -> int:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def current_stream() -> int:
    import torch

    return torch.cuda.current_stream().cuda_stream


def profile_step(fn):
    """Run ``fn()`` (which enqueues kernels eagerly) with per-kernel CUDA-event timing.
    Returns {label: (total_ms, launches)} in launch order."""
    lib = load()
    lib.nnp_profile_begin()
    fn()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.nnp_profile_report(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, ms, cnt = line.split()
        out[name] = (float(ms), int(cnt))
    return out
