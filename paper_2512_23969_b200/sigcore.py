"""Keys, signature layout and the public keygen / sign / verify API.

Drop-in for the reference's sigcore.py (sigcore.py:26-221): same names,
argument meaning, byte layouts and error behaviour, but every hash runs on
the B200 through the C-ABI (no CPU signing path exists in this package).

    sk  = sk_seed || sk_prf || pk_seed || pk_root
    pk  = pk_seed || pk_root
    sig = randomizer || fors_sig || d * (wots_sig || auth_path)

Batch entry points (``sign_batch``, ``verify_batch``, ``keygen_batch``) are
the native shape of the engine: one CUDA-graph launch signs a whole batch.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Sequence

from .engine import get_engine, get_multi_engine
from .errors import FormatError, UsageError
from .params import DerivedParams, compressions_per_signature, derive


@dataclass(frozen=True)
class PublicKey:
    pk_seed: bytes
    pk_root: bytes

    def to_bytes(self) -> bytes:
        return self.pk_seed + self.pk_root

    @classmethod
    def from_bytes(cls, data: bytes, p: DerivedParams) -> "PublicKey":
        p = derive(p)
        if len(data) != p.pk_bytes:
            raise FormatError(f"public key must be {p.pk_bytes} bytes, got {len(data)}")
        return cls(bytes(data[: p.n]), bytes(data[p.n:]))


@dataclass(frozen=True)
class SecretKey:
    sk_seed: bytes
    sk_prf: bytes
    pk_seed: bytes
    pk_root: bytes

    def to_bytes(self) -> bytes:
        return self.sk_seed + self.sk_prf + self.pk_seed + self.pk_root

    @classmethod
    def from_bytes(cls, data: bytes, p: DerivedParams) -> "SecretKey":
        p = derive(p)
        if len(data) != p.sk_bytes:
            raise FormatError(f"secret key must be {p.sk_bytes} bytes, got {len(data)}")
        n = p.n
        data = bytes(data)
        return cls(data[:n], data[n:2 * n], data[2 * n:3 * n], data[3 * n:])

    def public(self) -> PublicKey:
        return PublicKey(self.pk_seed, self.pk_root)


class SignContext:
    """Stand-in for the reference's HashContext handed out via ``ctx_out``
    (sigcore.py:166-168).

    ``compressions`` is the exact SHA-256 compression count the reference's
    default path records for this signature (hashes.py:117-159): the fixed
    per-stage terms of params.compressions_per_signature plus ``wots_steps``,
    the WOTS_Sign F steps the device counted while signing (the sum of the
    signed base-w digits over all layers).
    """

    def __init__(self, p: DerivedParams, msg_len: int, wots_steps: int):
        self.params = p
        self.wots_steps = int(wots_steps)
        self.compressions = int(compressions_per_signature(p, msg_len, digit_sum=self.wots_steps)["total"])


def _sk_of(sk) -> SecretKey:
    if isinstance(sk, SecretKey):
        return sk
    if hasattr(sk, "to_bytes") and hasattr(sk, "sk_seed"):
        return SecretKey(sk.sk_seed, sk.sk_prf, sk.pk_seed, sk.pk_root)
    raise UsageError("sk must be a SecretKey")


def _apply_overrides(eng, p, fusion, relax, selection) -> dict | None:
    """Map the reference's per-call layout knobs onto the engine config."""
    if fusion is None and relax is None and selection is None:
        return None
    before = eng.config(p.id)
    kw = {}
    if fusion is not None:
        # an explicit layout is run as given, whatever the batch size
        kw["fors_trees_per_set"] = int(fusion.trees_per_set)
        kw["fors_sets_fused"] = int(fusion.sets_fused)
        kw["fors_small_batch"] = 0
    if relax is not None:
        kw["fors_relax"] = bool(getattr(relax, "enabled", relax))
    if selection is not None:
        # reference backends (backends.py:201-257): "baseline" -> the native path;
        # "tuned" -> the path the on-device tuner chose for this kernel (the
        # configured one), or the fast path where the config says native
        var = {}
        for kernel in ("FORS_Sign", "TREE_Sign", "WOTS_Sign"):
            b = selection.get(kernel, p.id)
            tuned = str(getattr(b, "value", b)) == "tuned"
            var[kernel] = (before["variant"][kernel] or 1) if tuned else 0
        kw["variant"] = var
    eng.set_config(p.id, **kw)
    return before


def keygen(params: DerivedParams | str, seed: bytes | None = None) -> SecretKey:
    """Generate a keypair; seed is sk_seed || sk_prf || pk_seed (3n bytes) (sigcore.py:62-72)."""
    p = derive(params)
    if seed is None:
        seed = os.urandom(3 * p.n)
    if len(seed) != 3 * p.n:
        raise UsageError(f"seed must be {3 * p.n} bytes, got {len(seed)}")
    return SecretKey.from_bytes(get_engine().keygen_batch(p.id, [bytes(seed)])[0], p)


def keygen_batch(params: DerivedParams | str, seeds: Sequence[bytes]) -> list[SecretKey]:
    p = derive(params)
    return [SecretKey.from_bytes(b, p) for b in get_engine().keygen_batch(p.id, [bytes(s) for s in seeds])]


def sign(
    msg: bytes,
    sk: SecretKey,
    params: DerivedParams | str,
    *,
    opt_rand: bytes | None = None,
    oracle: bool = False,
    fusion=None,
    relax=None,
    workers: int = 1,
    selection=None,
    pure: bool = False,
    instrument=None,
    ctx_out: list | None = None,
) -> bytes:
    """Sign one message (sigcore.py:139-178); deterministic given (msg, sk, opt_rand).

    ``oracle``, ``workers``, ``pure`` and ``instrument`` select CPU execution
    shapes of the reference and do not change bytes; they are accepted for
    call compatibility.  ``fusion``/``relax``/``selection`` set the FORS
    layout and SHA-256 paths for this call.
    """
    return sign_batch([msg], sk, params, opt_rand=None if opt_rand is None else [opt_rand], fusion=fusion,
                      relax=relax, selection=selection, ctx_out=ctx_out)[0]


def sign_batch(
    msgs: Sequence[bytes],
    sk,
    params: DerivedParams | str,
    *,
    key_idx: Sequence[int] | None = None,
    opt_rand: Sequence[bytes] | None = None,
    fusion=None,
    relax=None,
    selection=None,
    ctx_out: list | None = None,
    devices: Sequence[int] | None = None,
) -> list[bytes]:
    """Sign a batch in one graph launch per device.  ``sk`` is one SecretKey or
    a list (then ``key_idx[i]`` picks message i's key; default key 0).
    ``devices`` (e.g. ``range(8)``) shards the batch by message over those
    GPUs (engine.MultiEngine); default: this process's device."""
    eng = get_engine() if devices is None else get_multi_engine(devices)
    return sign_on_engine(eng, msgs, sk, params, key_idx=key_idx, opt_rand=opt_rand, fusion=fusion, relax=relax,
                          selection=selection, ctx_out=ctx_out)


def sign_on_engine(
    eng,
    msgs: Sequence[bytes],
    sk,
    params: DerivedParams | str,
    *,
    key_idx: Sequence[int] | None = None,
    opt_rand: Sequence[bytes] | None = None,
    fusion=None,
    relax=None,
    selection=None,
    ctx_out: list | None = None,
) -> list[bytes]:
    """``sign_batch`` on a given engine (an ``Engine``, or any object with its
    lock / upload_keys / config / set_config / sign_batch methods)."""
    p = derive(params)
    keys = [_sk_of(k) for k in (sk if isinstance(sk, (list, tuple)) else [sk])]
    if not keys:
        raise UsageError("at least one secret key is required")
    for k in keys:
        if len(k.to_bytes()) != p.sk_bytes:
            raise UsageError(f"secret key must be {p.sk_bytes} bytes for {p.id}")
    if opt_rand is not None:
        opt_rand = list(opt_rand)
        if len(opt_rand) != len(msgs):
            raise UsageError("one opt_rand per message required")
        for o in opt_rand:
            if o is not None and len(o) != p.n:
                raise UsageError(f"opt_rand must be {p.n} bytes, got {len(o)}")
        if any(o is None for o in opt_rand):
            kk = list(key_idx) if key_idx is not None else [0] * len(msgs)
            opt_rand = [o if o is not None else keys[kk[i]].pk_seed for i, o in enumerate(opt_rand)]
    # the engine is process-wide: key table, per-call overrides, the sign and
    # the restore form one critical section, so concurrent callers (threads,
    # several GraphSigners) never sign under each other's keys or layout
    with eng.lock:
        eng.upload_keys(p.id, [k.to_bytes() for k in keys])
        before = _apply_overrides(eng, p, fusion, relax, selection)
        try:
            res = eng.sign_batch(p.id, [bytes(m) for m in msgs], key_idx=key_idx, opt_rand=opt_rand,
                                 counts=ctx_out is not None)
        finally:
            if before is not None:
                eng.set_config(p.id, **before)
    if ctx_out is None:
        return res
    sigs, steps = res
    for m, st in zip(msgs, steps):
        ctx_out.append(SignContext(p, len(m), st))
    return sigs


def verify(msg: bytes, sig: bytes, pk: PublicKey, params: DerivedParams | str) -> bool:
    """Recompute the FORS root and walk all d layers on the GPU (sigcore.py:181-221)."""
    p = derive(params)
    if len(sig) != p.sig_bytes:
        return False
    return verify_batch([msg], [sig], pk, p)[0]


def verify_batch(msgs: Sequence[bytes], sigs: Sequence[bytes], pk, params, *,
                 key_idx: Sequence[int] | None = None, devices: Sequence[int] | None = None) -> list[bool]:
    p = derive(params)
    pks = [k.to_bytes() if hasattr(k, "to_bytes") else bytes(k) for k in (pk if isinstance(pk, (list, tuple)) else [pk])]
    eng = get_engine() if devices is None else get_multi_engine(devices)
    return eng.verify_batch(p.id, pks, [bytes(m) for m in msgs], [bytes(s) for s in sigs], key_idx=key_idx)


def message_to_indices(mhash: bytes, p: DerivedParams) -> list[int]:
    """k log_t-bit chunks, least-significant bit first within each byte (sigcore.py:75-90)."""
    p = derive(p)
    assert len(mhash) * 8 >= p.k * p.log_t, "digest too short for index extraction"
    out, off = [], 0
    for _ in range(p.k):
        v = 0
        for j in range(p.log_t):
            v |= ((mhash[off >> 3] >> (off & 7)) & 1) << j
            off += 1
        out.append(v)
    return out


def signature_regions(p: DerivedParams) -> dict[str, tuple[int, int]]:
    """Byte ranges of the signature layout (sigcore.py:124-136)."""
    p = derive(p)
    regions = {"randomizer": (0, p.n)}
    off = p.n
    regions["fors"] = (off, off + p.fors_sig_bytes)
    off += p.fors_sig_bytes
    for layer in range(p.d):
        regions[f"wots[{layer}]"] = (off, off + p.wots_sig_bytes)
        off += p.wots_sig_bytes
        regions[f"auth[{layer}]"] = (off, off + p.subtree_height * p.n)
        off += p.subtree_height * p.n
    assert off == p.sig_bytes
    return regions
