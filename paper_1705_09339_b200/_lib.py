"""ctypes binding of the C-ABI in include/cog_b200.h (libcog_b200.so).

The shared library is built in-tree by ``build_extension()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
library is missing or cannot be loaded, every entry point raises
``CudaError`` -- the engine never silently runs anything else.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from pathlib import Path

from .errors import CudaError

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SO_PATH = PKG / "libcog_b200.so"
SOURCES = [PKG / "csrc" / "cog_kernels.cu"]
# every header the translation unit includes (a stale .so after editing one
# of them would silently run old code)
HEADERS = sorted((PKG / "csrc").glob("*.cuh")) + [ROOT / "include" / "cog_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # binary64 decisions must not be contracted into FMAs (parity contract)
    "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared",
]

COG_EINVAL = -1
COG_EUNSUPPORTED = -2

_lock = threading.Lock()
_lib = None


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def build_extension(force: bool = False, verbose: bool = False,
                    defines: tuple = ()) -> Path:
    """Compile libcog_b200.so in-tree if it is missing or stale.  `defines`
    (NAME=VALUE build-time tuning macros, tools/ab_build.sh) force a
    rebuild."""
    newest = max(p.stat().st_mtime for p in SOURCES + HEADERS)
    if (not force and not defines and SO_PATH.exists()
            and SO_PATH.stat().st_mtime >= newest):
        return SO_PATH
    tmp = SO_PATH.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines],
           "-I", str(ROOT / "include"), "-o", str(tmp),
           *[str(s) for s in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise CudaError("nvcc failed building libcog_b200.so:\n" + res.stderr)
    if verbose:
        print(res.stderr)
    os.replace(tmp, SO_PATH)
    return SO_PATH


# ------------------------------------------------------------------ structs


class Geom(ctypes.Structure):
    _fields_ = [
        ("total_pixels", ctypes.c_int64),
        ("height", ctypes.c_int32), ("width", ctypes.c_int32),
        ("depth", ctypes.c_int32), ("k", ctypes.c_int32),
        ("stride", ctypes.c_int32), ("n_groups", ctypes.c_int32),
        ("streams", ctypes.c_int32), ("state_f64", ctypes.c_int32),
        ("row0", ctypes.c_int32), ("pad_", ctypes.c_int32),
    ]


class Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in (
        "learning_rate", "match_lambda", "background_threshold",
        "variance_floor", "initial_variance", "chp_epsilon",
        "confidence_threshold", "prior_floor", "rate_floor",
        "illumination_fraction")] + [
        ("weights", ctypes.c_double * 9)] + [
        (n, ctypes.c_int32) for n in (
            "saturation_frames", "sleep_frames", "sampling_on", "grouping_on",
            "rate_scaling_on", "chp_on", "literal_conf", "compat",
            "exact_group_sums", "variant")]


# cog_params.variant: which step kernel (a parity knob; 0 = automatic)
VARIANTS = {"auto": 0, "general": 1, "lean": 2, "tiles": 3}


class State(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "mix", "meta", "dyn", "streak", "hits", "table", "peak", "tabq",
        "cls", "gid", "g_mu", "g_var", "g_members", "accum", "sync",
        "deepq", "deeprho", "hitq")]


MAX_RANKS = 16


class Peers(ctypes.Structure):
    """cog_peers: the peer mailboxes of a row-band shard (cog_step_p2p)."""
    _fields_ = [("n_ranks", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("seq", ctypes.c_uint64),
                ("mailbox", ctypes.c_void_p * MAX_RANKS)]


class RefState(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "mu", "var", "w", "count", "mid", "ref", "chp", "label", "active",
        "waking", "streak", "clock", "hits")]


_P = ctypes.c_void_p
_SIGS = {
    "cog_accum_words": (ctypes.c_int64, [ctypes.c_int32, ctypes.c_int32]),
    "cog_mix_elems": (ctypes.c_int64, [ctypes.c_int32]),
    "cog_tabq_elems": (ctypes.c_int64, [_P]),
    "cog_tabq_build": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "cog_deepq_slots": (ctypes.c_int64, [ctypes.c_int32, ctypes.c_int64]),
    "cog_prior_build": (ctypes.c_int, [
        _P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, _P, _P,
        ctypes.c_int32, _P, _P, _P, ctypes.c_double, ctypes.c_double,
        ctypes.c_double, _P, _P, _P]),
    "cog_gmm_warmup": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_int32, _P, _P,
                                      _P]),
    "cog_set_levels": (ctypes.c_int, [_P, _P, _P]),
    "cog_step": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P,
                                ctypes.c_int64, ctypes.c_int32,
                                ctypes.c_int32, _P]),
    "cog_finalize": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_int64, _P]),
    "cog_mailbox_words": (ctypes.c_int64, [ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_int32]),
    "cog_step_p2p": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P,
                                    ctypes.c_int64, ctypes.c_int32,
                                    ctypes.c_int32, _P, _P]),
    "cog_finalize_p2p": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_int64, _P,
                                        _P]),
    "cog_apply_pending": (ctypes.c_int, [_P, _P, _P, ctypes.c_int32, _P]),
    "cog_baseline_frame": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "cog_export_state": (ctypes.c_int, [_P, _P, _P, _P]),
    "cog_import_state": (ctypes.c_int, [_P, _P, _P, _P]),
    "cog_step_host": (ctypes.c_int, [_P] * 11 + [ctypes.c_int64,
                                                ctypes.c_int32] + [_P] * 5),
    "cog_seq_sums": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_int32, _P,
                                    ctypes.c_int32, _P, ctypes.c_int32, _P,
                                    _P, _P, _P]),
    "cog_far_step": (ctypes.c_int, [_P, ctypes.c_int64, _P, ctypes.c_int32,
                                    _P, _P, _P]),
    "cog_confusion": (ctypes.c_int, [_P, _P, ctypes.c_int64, _P, _P]),
    "cog_pool_sums": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_int64, _P, ctypes.c_int32,
                                     _P, _P]),
    "cog_kmeans_assign": (ctypes.c_int, [_P, ctypes.c_int64, _P,
                                         ctypes.c_int32, _P, _P, _P]),
    "cog_event_create": (ctypes.c_void_p, []),
    "cog_event_destroy": (ctypes.c_int, [_P]),
    "cog_event_sync": (ctypes.c_int, [_P]),
    "cog_event_query": (ctypes.c_int, [_P]),
    "cog_version": (ctypes.c_char_p, []),
}

EXPORTED = tuple(_SIGS)


def load(path: Path | None = None):
    """Load (building first if needed) and return the ctypes library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        so = Path(path or os.environ.get("COG_LIB") or SO_PATH)
        if not so.exists():
            try:
                build_extension()
            except (OSError, CudaError) as exc:
                raise CudaError(f"CUDA extension {so} is missing and could "
                                f"not be built: {exc}") from exc
        try:
            lib = ctypes.CDLL(str(so))
        except OSError as exc:
            raise CudaError(f"cannot load CUDA extension {so}: {exc}") from exc
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    if rc == COG_EINVAL:
        raise CudaError(f"{what}: invalid arguments")
    if rc == COG_EUNSUPPORTED:
        raise CudaError(f"{what}: unsupported geometry / configuration")
    raise CudaError(f"{what}: CUDA error {rc}")


def ref(obj) -> ctypes.c_void_p:
    return ctypes.cast(ctypes.pointer(obj), ctypes.c_void_p)
