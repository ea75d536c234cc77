"""ctypes binding of libsfdt_b200.so (include/sfdt.h).

The product path has exactly one implementation: the sm_100a kernels in this
library.  There is no CPU fallback -- if the library is missing or no CUDA
device is present, calls fail loudly.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SFDT_LIB") or os.path.join(_HERE, "libsfdt_b200.so")

SFDT_ST_NITER = 0
SFDT_ST_FULL_SUCCESS = 1
SFDT_ST_NENTRIES = 2
SFDT_ST_NUNRESOLVED = 3
SFDT_ST_NDUP = 4
SFDT_ST_SYNDROMES = 5
SFDT_ST_FFT_SAMPLES = 6
SFDT_ST_ITER0 = 8
SFDT_ST_PER_SIGNAL = 32
SFDT_C128, SFDT_C64 = 0, 1

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_int = ctypes.c_int
_dbl = ctypes.c_double


class Tuning(ctypes.Structure):
    """sfdt_tuning (include/sfdt.h): A/B switches of measured design decisions."""
    _fields_ = [(name, _i32) for name in (
        "fft_split", "gen_dedup", "gen_svd_closed", "gen_mf_small", "gen_mf_list", "gen_warp",
        "gen_split_a", "gen_prune_lanes", "gen_deal", "decode_coop", "latency_path", "gen_window")]


class ExactArgs(ctypes.Structure):
    _fields_ = [
        ("x", _vp), ("x_dtype", _i32), ("batch", _i64), ("n", _i64),
        ("d", _i64), ("a_max", _i32), ("iterative", _i32), ("zero_threshold", _dbl),
        ("twiddles", _vp),
        ("entry_offsets", _vp), ("locs", _vp), ("vals", _vp), ("entry_cap", _i64),
        ("unres_offsets", _vp), ("unres_bins", _vp), ("unres_cap", _i64),
        ("dup_locs", _vp), ("dup_offsets", _vp), ("dup_cap", _i64),
        ("stats", _vp), ("rms", _vp),
        ("aux_stream", _vp), ("chunk_signals", _i64), ("rms_in", _vp),
        ("ev_stream_begin", _vp), ("ev_stream_end", _vp), ("tuning", _vp), ("kernel_launches", _i32),
    ]


SFDT_GS_NENTRIES = 0
SFDT_GS_HIST0 = 1
SFDT_GS_NVOTED = 6
SFDT_GS_RANKDEF = 7
SFDT_GS_CLASS0 = 8
SFDT_GS_PER_SIGNAL = 16


class GeneralArgs(ctypes.Structure):
    _fields_ = [
        ("x", _vp), ("x_dtype", _i32), ("batch", _i64), ("n", _i64),
        ("k", _i64), ("d", _i64), ("a_max", _i32), ("r_eff", _i32),
        ("keep_per_collision", _i32), ("prune", _i32), ("zero_vote_rtol", _dbl),
        ("shifts", _vp), ("shift_stride", _i64), ("base_phi", _vp), ("phi_stride", _i64),
        ("twiddles", _vp),
        ("entry_offsets", _vp), ("locs", _vp), ("vals", _vp), ("entry_cap", _i64),
        ("stats", _vp), ("votes", _vp), ("singular_values", _vp),
        ("ev_fft_begin", _vp), ("ev_fft_end", _vp),
        ("ev_vote_end", _vp), ("ev_prune_end", _vp), ("ev_pursuit_end", _vp),
        ("aux_stream", _vp), ("tuning", _vp),
        ("kernel_launches", _i32),
    ]


# every symbol include/sfdt.h declares (tests check the export list)
EXPORTS = {
    "sfdt_strerror": (ctypes.c_char_p, [_int]),
    "sfdt_version": (_int, []),
    "sfdt_default_tuning": (None, [ctypes.POINTER(Tuning)]),
    "sfdt_last_cuda_error": (ctypes.c_char_p, []),
    "sfdt_fft_twiddles": (_int, [_i64, _int, _vp]),
    "sfdt_fft_radix2": (_int, [_vp, _vp, _i64, _i64, _int, _vp, _vp]),
    "sfdt_hankel_solve": (_int, [_vp, _i64, _i64, _int, _vp, _vp, _vp]),
    "sfdt_poly_roots": (_int, [_vp, _i64, _int, _vp, _vp]),
    "sfdt_vandermonde_solve": (_int, [_vp, _vp, _i64, _int, _i64, _vp, _vp, _vp]),
    "sfdt_prune_eval": (_int, [_vp, _vp, _i64, _int, _i64, _i64, _vp, _vp]),
    "sfdt_hankel_singular_values": (_int, [_vp, _i64, _i64, _int, _vp, _vp]),
    "sfdt_exact_caps": (_int, [ctypes.POINTER(ExactArgs), ctypes.POINTER(_i64),
                               ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "sfdt_exact_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(ExactArgs)]),
    "sfdt_exact_solve": (_int, [ctypes.POINTER(ExactArgs), _vp, ctypes.c_size_t, _vp]),
    "sfdt_estimate_collisions_workspace_bytes": (ctypes.c_size_t, [_i64]),
    "sfdt_estimate_collisions": (_int, [_vp, _i64, _i64, _i64, _int, _i64, _dbl, _vp, _vp, _vp,
                                        ctypes.c_size_t, _vp]),
    "sfdt_general_caps": (_int, [ctypes.POINTER(GeneralArgs), ctypes.POINTER(_i64)]),
    "sfdt_general_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(GeneralArgs)]),
    "sfdt_general_solve": (_int, [ctypes.POINTER(GeneralArgs), _vp, ctypes.c_size_t, _vp]),
    "sfdt_graph_submit": (_int, [_vp, _vp, ctypes.c_size_t, _vp, _vp, _vp, _vp]),
    "sfdt_downsample": (_int, [_vp, _i32, _i64, _i64, _i64, _vp, _i32, _vp, _vp]),
    "sfdt_aliased_values_workspace_bytes": (ctypes.c_size_t, [_i64, _i64, _i64, _i32]),
    "sfdt_aliased_values": (_int, [_vp, _i32, _i64, _i64, _i64, _vp, _i32, _vp, _vp, _vp,
                                   ctypes.c_size_t, _vp]),
    "sfdt_direct_dft": (_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "sfdt_rms_workspace_bytes": (ctypes.c_size_t, [_i64, _i64]),
    "sfdt_rms": (_int, [_vp, _i32, _i64, _i64, _vp, _vp, ctypes.c_size_t, _vp]),
    "sfdt_decode_bins": (_int, [_vp, _i64, _i64, _int, _i64, _i64, _vp, _int, _vp, _vp, _vp, _vp,
                                _vp, _vp, _vp, _vp, _vp]),
    "sfdt_poly_residuals": (_int, [_vp, _vp, _i64, _int, _vp, _vp]),
    "sfdt_reconstruct_syndromes": (_int, [_vp, _vp, _i64, _int, _int, _vp, _vp]),
    "sfdt_sensing_matrix": (_int, [_i64, _i64, _i64, _vp, _int, _vp, _i64, _vp, _vp]),
    "sfdt_prune_columns": (_int, [_vp, _i64, _i64, _vp, _int, _int, _i64, _i64, _int, _vp, _i64,
                                  _vp, _int, _int, _vp, _vp, _i64, _vp]),
    "sfdt_subspace_pursuit": (_int, [_vp, _vp, _i64, _int, _int, _int, _int, _vp, _vp, _vp]),
}

SFDT_DB_OK, SFDT_DB_NEAR_SINGULAR, SFDT_DB_DEGENERATE, SFDT_DB_ILL_CONDITIONED, SFDT_DB_ZERO_ROOT = range(5)

_lib = None

# ------------------------------------------------------------ A/B switches
# The library reads no environment: its design switches arrive as an
# sfdt_tuning with every solve.  Defaults are the measured-best decisions;
# `tuning(...)` overrides them for a block of calls (tests), and the SFDT_*
# environment variables of the experiment scripts (tools/*.sh) are read ONCE,
# at the first solve, into the process defaults.
TUNING_DEFAULTS = dict(fft_split=0, gen_dedup=1, gen_svd_closed=1, gen_mf_small=1, gen_mf_list=0,
                       gen_warp=-1, gen_split_a=3, gen_prune_lanes=0, gen_deal=8, gen_overlap=1, decode_coop=-1, latency_path=-1, gen_window=-1)
_ENV = None
_local = threading.local()


def _env_overrides() -> dict:
    global _ENV
    if _ENV is None:
        e, o = os.environ.get, {}
        if e("SFDT_FFT_SPLIT") is not None:
            o["fft_split"] = int(e("SFDT_FFT_SPLIT"))
        if e("SFDT_FFT_PIPE") == "0":
            o["fft_split"] = 1
        for var, key in (("SFDT_GEN_DEDUP", "gen_dedup"), ("SFDT_GEN_MF_SMALL", "gen_mf_small"),
                         ("SFDT_GEN_MF_LIST", "gen_mf_list"), ("SFDT_GEN_WARP", "gen_warp"),
                         ("SFDT_GEN_SPLIT", "gen_split_a"), ("SFDT_GEN_PRUNE_LANES", "gen_prune_lanes"),
                         ("SFDT_GEN_DEAL", "gen_deal"), ("SFDT_GEN_OVERLAP", "gen_overlap"),
                         ("SFDT_DECODE_COOP", "decode_coop"), ("SFDT_LATENCY_PATH", "latency_path"),
                         ("SFDT_GEN_WINDOW", "gen_window")):
            if e(var) is not None:
                o[key] = int(e(var))
        if e("SFDT_GEN_SVD") is not None:
            o["gen_svd_closed"] = 0 if e("SFDT_GEN_SVD").startswith("j") else 1
        _ENV = o
    return _ENV


def current_tuning() -> dict:
    t = dict(TUNING_DEFAULTS)
    t.update(_env_overrides())
    for over in getattr(_local, "stack", []):
        t.update(over)
    return t


@contextlib.contextmanager
def tuning(**overrides):
    """Override design switches for the solves issued inside the block
    (keys of TUNING_DEFAULTS), e.g. ``with tuning(gen_svd_closed=0): ...``."""
    bad = set(overrides) - set(TUNING_DEFAULTS)
    if bad:
        raise KeyError(f"unknown tuning keys {sorted(bad)}")
    stack = getattr(_local, "stack", None)
    if stack is None:
        stack = _local.stack = []
    stack.append(overrides)
    try:
        yield
    finally:
        stack.pop()


def tuning_struct(t: dict | None = None) -> "Tuning":
    t = current_tuning() if t is None else t
    return Tuning(**{name: int(t[name]) for name, _ in Tuning._fields_})


class SfdtError(RuntimeError):
    pass


def load():
    """Load (and type) the library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} missing: build it with `python -m paper_1407_8315_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str):
    if rc != 0:
        msg = load().sfdt_strerror(rc).decode()
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        if rc == -2:
            msg += f" [{load().sfdt_last_cuda_error().decode()}]"
        raise SfdtError(f"{what}: {msg} ({rc})")
