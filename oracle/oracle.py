"""ctypes view of the C oracle (oracle/hs_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module, and only as the checker / the timed CPU reference.  The
product package (paper_2512_23969_b200) never imports it.

Every wrapper mirrors a function of the reference package (paths relative to
the reference's pkg/src/herosign/):

    thash          hashes.py:124-137      prf        hashes.py:139-150
    prf_msg        hashes.py:152-165      h_msg      hashes.py:175-191
    indices        sigcore.py:75-90       chain_lengths  wots.py:33-39
    wots_gen_leaf  wots.py:119-143        tree_layer vexec.py:492-551
    fors_sign      oracle.py:113-146      wots_sign  wots.py:68-82
    keygen         sigcore.py:62-72       sign       sigcore.py:139-178
    verify         sigcore.py:181-221
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libhs_oracle.so"
_SETS = {"128f": 0, "192f": 1, "256f": 2}
_FIELDS = (
    "n h d log_t k w lg_w len1 len2 wots_len hp leaves t fors_msg_bytes tree_bits "
    "tree_bytes leaf_bits leaf_bytes digest_bytes wots_sig_bytes fors_sig_bytes "
    "ht_sig_bytes sig_bytes"
).split()

_lib = None


def build() -> Path:
    """Compile the oracle with its Makefile (gcc only; seconds)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(_LIB_PATH))
        u8p = ctypes.c_char_p
        _lib.hso_sign.argtypes = [ctypes.c_int, u8p, u8p, ctypes.c_size_t, u8p,
                                  ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]
        _lib.hso_verify.argtypes = [ctypes.c_int, u8p, u8p, ctypes.c_size_t, u8p, ctypes.c_size_t]
        _lib.hso_sign_many.argtypes = [
            ctypes.c_int, ctypes.c_int, u8p, ctypes.c_void_p, u8p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_uint32, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64),
        ]
        _lib.hso_wots_gen_leaf.argtypes = [ctypes.c_int, u8p, u8p, ctypes.c_uint32, ctypes.c_uint64,
                                           ctypes.c_uint32, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]
        _lib.hso_tree_layer.argtypes = [ctypes.c_int, u8p, u8p, ctypes.c_uint32, ctypes.c_uint64,
                                        ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]
        _lib.hso_fors_sign.argtypes = [ctypes.c_int, u8p, u8p, ctypes.c_uint64, ctypes.c_uint32,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib.hso_wots_sign.argtypes = [ctypes.c_int, u8p, u8p, ctypes.c_uint32, ctypes.c_uint64,
                                       ctypes.c_uint32, u8p, ctypes.c_void_p]
        _lib.hso_h_msg.argtypes = [ctypes.c_int, u8p, u8p, u8p, u8p, ctypes.c_size_t, ctypes.c_void_p,
                                   ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32)]
        _lib.hso_prf_msg.argtypes = [ctypes.c_int, u8p, u8p, u8p, ctypes.c_size_t, ctypes.c_void_p]
        _lib.hso_thash.argtypes = [ctypes.c_int, u8p, u8p, u8p, ctypes.c_size_t, ctypes.c_void_p]
        _lib.hso_prf.argtypes = [ctypes.c_int, u8p, u8p, ctypes.c_void_p]
        _lib.hso_sha256.argtypes = [u8p, ctypes.c_size_t, ctypes.c_void_p]
        _lib.hso_compress.argtypes = [ctypes.c_void_p, u8p]
    return _lib


def set_index(set_id: str) -> int:
    return _SETS[set_id]


def params(set_id: str) -> dict:
    out = (ctypes.c_int * 32)()
    cnt = lib().hso_params(_SETS[set_id], out)
    return dict(zip(_FIELDS, out[:cnt]))


def force_scalar(on: bool) -> None:
    lib().hso_force_scalar(1 if on else 0)


def shani_active() -> bool:
    return bool(lib().hso_shani_active())


def sha256(data: bytes) -> bytes:
    out = ctypes.create_string_buffer(32)
    lib().hso_sha256(data, len(data), out)
    return out.raw


def compress(state: tuple, block: bytes) -> tuple:
    st = (ctypes.c_uint32 * 8)(*state)
    lib().hso_compress(st, block)
    return tuple(st)


def thash(set_id: str, pk_seed: bytes, adrs: bytes, msg: bytes) -> bytes:
    n = params(set_id)["n"]
    out = ctypes.create_string_buffer(32)
    lib().hso_thash(_SETS[set_id], pk_seed, adrs, msg, len(msg), out)
    return out.raw[:n]


def prf(set_id: str, sk_seed: bytes, adrs: bytes) -> bytes:
    n = params(set_id)["n"]
    out = ctypes.create_string_buffer(32)
    lib().hso_prf(_SETS[set_id], sk_seed, adrs, out)
    return out.raw[:n]


def prf_msg(set_id: str, sk_prf: bytes, opt_rand: bytes, msg: bytes) -> bytes:
    n = params(set_id)["n"]
    out = ctypes.create_string_buffer(32)
    lib().hso_prf_msg(_SETS[set_id], sk_prf, opt_rand, msg, len(msg), out)
    return out.raw[:n]


def h_msg(set_id: str, R: bytes, pk_seed: bytes, pk_root: bytes, msg: bytes):
    p = params(set_id)
    mh = ctypes.create_string_buffer(64)
    tree = ctypes.c_uint64()
    leaf = ctypes.c_uint32()
    lib().hso_h_msg(_SETS[set_id], R, pk_seed, pk_root, msg, len(msg), mh, ctypes.byref(tree), ctypes.byref(leaf))
    return mh.raw[: p["fors_msg_bytes"]], tree.value, leaf.value


def message_to_indices(set_id: str, mhash: bytes) -> list[int]:
    out = (ctypes.c_uint32 * 64)()
    k = lib().hso_message_to_indices(_SETS[set_id], mhash, out)
    return list(out[:k])


def chain_lengths(set_id: str, msg_n: bytes) -> list[int]:
    out = (ctypes.c_uint32 * 80)()
    m = lib().hso_chain_lengths(_SETS[set_id], msg_n, out)
    return list(out[:m])


def wots_gen_leaf(set_id, pk_seed, sk_seed, layer, tree, leaf_idx):
    n = params(set_id)["n"]
    out = ctypes.create_string_buffer(32)
    comps = ctypes.c_uint64()
    lib().hso_wots_gen_leaf(_SETS[set_id], pk_seed, sk_seed, layer, tree, leaf_idx, out, ctypes.byref(comps))
    return out.raw[:n], comps.value


def tree_layer(set_id, pk_seed, sk_seed, layer, tree, leaf_idx):
    p = params(set_id)
    root = ctypes.create_string_buffer(32)
    auth = ctypes.create_string_buffer(p["hp"] * p["n"])
    lib().hso_tree_layer(_SETS[set_id], pk_seed, sk_seed, layer, tree, leaf_idx, root, auth)
    return root.raw[: p["n"]], auth.raw


def fors_sign(set_id, pk_seed, sk_seed, tree, leaf_idx, indices):
    p = params(set_id)
    idx = (ctypes.c_uint32 * len(indices))(*indices)
    sig = ctypes.create_string_buffer(p["fors_sig_bytes"])
    pk = ctypes.create_string_buffer(32)
    lib().hso_fors_sign(_SETS[set_id], pk_seed, sk_seed, tree, leaf_idx, idx, sig, pk)
    return sig.raw, pk.raw[: p["n"]]


def wots_sign(set_id, pk_seed, sk_seed, layer, tree, keypair, msg_n):
    p = params(set_id)
    sig = ctypes.create_string_buffer(p["wots_sig_bytes"])
    lib().hso_wots_sign(_SETS[set_id], pk_seed, sk_seed, layer, tree, keypair, msg_n, sig)
    return sig.raw


def keygen(set_id: str, seed: bytes) -> bytes:
    p = params(set_id)
    sk = ctypes.create_string_buffer(4 * p["n"])
    lib().hso_keygen(_SETS[set_id], seed, sk)
    return sk.raw


def sign(set_id: str, sk: bytes, msg: bytes, opt_rand: bytes | None = None) -> bytes:
    p = params(set_id)
    sig = ctypes.create_string_buffer(p["sig_bytes"])
    comps = ctypes.c_uint64()
    lib().hso_sign(_SETS[set_id], sk, msg, len(msg), opt_rand, sig, ctypes.byref(comps))
    return sig.raw


def verify(set_id: str, pk: bytes, msg: bytes, sig: bytes) -> bool:
    return bool(lib().hso_verify(_SETS[set_id], pk, msg, len(msg), sig, len(sig)))


def sign_many(set_id: str, sks: bytes, key_idx, msgs: list[bytes], opt_rands: bytes | None = None,
              threads: int | None = None) -> tuple[list[bytes], int]:
    """Sign every message on `threads` host threads; returns (sigs, compressions)."""
    p = params(set_id)
    count = len(msgs)
    offs = (ctypes.c_uint64 * (count + 1))()
    acc = 0
    for i, m in enumerate(msgs):
        offs[i] = acc
        acc += len(m)
    offs[count] = acc
    blob = b"".join(msgs)
    kidx = None
    if key_idx is not None:
        kidx = (ctypes.c_uint32 * count)(*key_idx)
    out = ctypes.create_string_buffer(count * p["sig_bytes"])
    comps = ctypes.c_uint64()
    lib().hso_sign_many(_SETS[set_id], threads or os.cpu_count() or 1, sks, kidx, blob, offs, opt_rands,
                        count, out, ctypes.byref(comps))
    sb = p["sig_bytes"]
    raw = out.raw
    return [raw[i * sb:(i + 1) * sb] for i in range(count)], comps.value
