"""ctypes binding of libherosign_b200.so (C-ABI: include/herosign_b200.h).

The shared library is built in-tree by ``build_native()`` (nvcc, sm_100a) and
loaded from this package directory.  There is no fallback: if the library is
missing or no CUDA device is visible, every engine call raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

from .errors import ConfigError, FormatError, HeroSignError, UsageError

PKG_DIR = Path(__file__).resolve().parent
# HERO_SIGN_LIB selects another build of the library (tools/variant_sweep.py)
LIB_PATH = Path(os.environ["HERO_SIGN_LIB"]) if os.environ.get("HERO_SIGN_LIB") else PKG_DIR / "libherosign_b200.so"
CSRC = PKG_DIR / "csrc"

HS_OK = 0
HS_E_USAGE = -1
HS_E_FORMAT = -2
HS_E_CONFIG = -3
HS_E_NOKEYS = -4
HS_E_CUDA = -10

EXPORTS = (
    "hs_open", "hs_close", "hs_last_error", "hs_device_info", "hs_params", "hs_config_get", "hs_config_set",
    "hs_fors_smem_bytes", "hs_keys_upload", "hs_keygen_batch", "hs_sign_batch", "hs_sign_batch_ex", "hs_verify_batch",
    "hs_stage", "hs_run", "hs_sync", "hs_fetch", "hs_timings", "hs_bench_run", "hs_launch_count", "hs_launch_stats", "hs_variants", "hs_batch_info", "hs_tune",
    "hs_host_alloc", "hs_host_free",
)


class SetConfig(ctypes.Structure):
    """hs_set_config (include/herosign_b200.h)."""

    _fields_ = [
        ("fors_trees_per_set", ctypes.c_int32),
        ("fors_sets_fused", ctypes.c_int32),
        ("fors_relax", ctypes.c_int32),
        ("variant", ctypes.c_int32 * 4),
        ("use_graph", ctypes.c_int32),
        ("chunk", ctypes.c_int32),
        ("wots_from_tree", ctypes.c_int32),
        ("streams", ctypes.c_int32),
        ("shared_layers", ctypes.c_int32),
        ("shared_auto", ctypes.c_int32),
        ("fors_cta_levels", ctypes.c_int32),
        ("tree_split", ctypes.c_int32),
        ("overlap", ctypes.c_int32),
        ("fors_small_batch", ctypes.c_int32),
        ("tree_small_batch", ctypes.c_int32),
    ]


_lib = None


def build_native(jobs: int | None = None) -> Path:
    """Compile the CUDA library for sm_100a with its Makefile (no GPU needed).

    The 22 objects (3 sets x 6 SHA-256 paths + per-set glue + host runtime)
    build in parallel, one job per host core by default."""
    jobs = jobs or max(4, min(24, os.cpu_count() or 4))
    subprocess.run(["make", "-s", "-j", str(jobs), "-C", str(CSRC)], check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise HeroSignError(
            f"{LIB_PATH.name} is not built; run paper_2512_23969_b200._lib.build_native() "
            "(or __graft_entry__.build())"
        )
    L = ctypes.CDLL(str(LIB_PATH))
    vp, u8p, i32, u32, i64 = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_int64
    sig = {
        "hs_open": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(vp)]),
        "hs_close": (None, [vp]),
        "hs_last_error": (ctypes.c_char_p, [vp]),
        "hs_device_info": (ctypes.c_int, [vp] + [ctypes.POINTER(i32)] * 4),
        "hs_params": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(i32), ctypes.c_int]),
        "hs_config_get": (ctypes.c_int, [vp, ctypes.c_int, ctypes.POINTER(SetConfig)]),
        "hs_config_set": (ctypes.c_int, [vp, ctypes.c_int, ctypes.POINTER(SetConfig)]),
        "hs_fors_smem_bytes": (i64, [ctypes.c_int, i32, i32, i32]),
        "hs_keys_upload": (ctypes.c_int, [vp, ctypes.c_int, u8p, u32]),
        "hs_keygen_batch": (ctypes.c_int, [vp, ctypes.c_int, u8p, u32, u8p]),
        "hs_sign_batch": (ctypes.c_int, [vp, ctypes.c_int, u8p, vp, vp, u8p, u32, u8p]),
        "hs_sign_batch_ex": (ctypes.c_int, [vp, ctypes.c_int, u8p, vp, vp, u8p, u32, u8p, vp]),
        "hs_verify_batch": (ctypes.c_int, [vp, ctypes.c_int, u8p, u32, u8p, vp, vp, u8p, u32, u8p]),
        "hs_stage": (ctypes.c_int, [vp, ctypes.c_int, u8p, vp, vp, u8p, u32]),
        "hs_run": (ctypes.c_int, [vp, ctypes.c_int, u32, ctypes.c_int]),
        "hs_sync": (ctypes.c_int, [vp]),
        "hs_fetch": (ctypes.c_int, [vp, ctypes.c_int, u32, u32, u8p]),
        "hs_timings": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_float), ctypes.c_int]),
        "hs_bench_run": (ctypes.c_int, [vp, ctypes.c_int, u32, i32, ctypes.c_int, ctypes.c_uint64,
                                        ctypes.POINTER(ctypes.c_float)]),
        "hs_launch_count": (i64, [vp]),
        "hs_launch_stats": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_int]),
        "hs_variants": (ctypes.c_int, [ctypes.POINTER(i32), ctypes.c_int]),
        "hs_batch_info": (ctypes.c_int, [vp, ctypes.c_int, ctypes.POINTER(i32), ctypes.c_int]),
        "hs_tune": (ctypes.c_int, [vp, ctypes.c_int, u32, i32, i32, ctypes.c_char_p, ctypes.c_size_t]),
        "hs_host_alloc": (vp, [ctypes.c_size_t]),
        "hs_host_free": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def variant_names() -> tuple[str, ...]:
    """Names of the SHA-256 paths compiled into the loaded library (hs_variants):
    ("native", "fast", "mx<mask>[p<order>]", ...), indexed by hs_set_config.variant id."""
    buf = (ctypes.c_int32 * 64)()
    n = lib().hs_variants(buf, 64)
    return ("native", "fast") + tuple(f"mx{buf[i] & 255}" + (f"p{buf[i] >> 8}" if buf[i] >> 8 else "")
                                      for i in range(n - 2))


def check(handle, rc: int, what: str) -> None:
    if rc == HS_OK:
        return
    msg = lib().hs_last_error(handle) if handle else b""
    text = f"{what}: {msg.decode(errors='replace') if msg else 'error'} (rc={rc})"
    if rc in (HS_E_USAGE, HS_E_NOKEYS):
        raise UsageError(text)
    if rc == HS_E_FORMAT:
        raise FormatError(text)
    if rc == HS_E_CONFIG:
        raise ConfigError(text)
    raise HeroSignError(text)


def default_device() -> int:
    for var in ("HEROSIGN_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(var)
        if v is not None and v.strip().isdigit():
            return int(v)
    return 0
