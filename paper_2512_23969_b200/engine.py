"""Engine: one handle per B200, wrapping the C-ABI (include/herosign_b200.h).

This is the stage-level replacement for the reference's signer objects
(GraphSigner batchgraph.py:245-353 and the sign path sigcore.py:139-178):
a batch of messages goes host -> device once, is signed by one CUDA-graph
launch (msg_prep -> {FORS_Sign -> T_k} || TREE_Sign -> WOTS_Sign) and comes
back as contiguous signature bytes.
"""

from __future__ import annotations

import ctypes
import threading
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from .errors import HeroSignError, UsageError
from .params import SET_INDEX, derive

KERNELS = ("FORS_Sign", "TREE_Sign", "WOTS_Sign", "host")  # hs_set_config.variant order


def variants() -> tuple[str, ...]:
    """SHA-256 arithmetic paths compiled into the library, by variant id (csrc/hs_variants.h)."""
    return _lib.variant_names()


def _u8ptr(buf):
    """Address (int) of a host buffer for a c_void_p argument, or None.  The
    caller keeps `buf` alive across the C call."""
    if buf is None:
        return None
    if isinstance(buf, int):
        return buf
    if isinstance(buf, np.ndarray):
        return buf.ctypes.data
    if isinstance(buf, bytes):
        return ctypes.cast(ctypes.c_char_p(buf), ctypes.c_void_p).value
    if isinstance(buf, (bytearray, memoryview)):
        return ctypes.addressof((ctypes.c_char * len(buf)).from_buffer(buf))
    raise UsageError(f"unsupported buffer type {type(buf).__name__}")


def _offsets(offs, count: int) -> np.ndarray:
    """offs as a contiguous uint64 array of at least count + 1 entries (the C
    side reads exactly count + 1)."""
    o = np.ascontiguousarray(offs, dtype=np.uint64)
    if o.ndim != 1 or o.shape[0] < count + 1:
        raise UsageError(f"offsets must hold count + 1 = {count + 1} entries, got {o.shape}")
    return o


def _key_index(key_idx, count: int) -> np.ndarray | None:
    if key_idx is None:
        return None
    k = np.ascontiguousarray(key_idx, dtype=np.uint32)
    if k.ndim != 1 or k.shape[0] < count:
        raise UsageError(f"key_idx must hold one entry per message ({count}), got {k.shape}")
    return k


def pack_messages(msgs: Sequence[bytes]) -> tuple[bytes, np.ndarray]:
    offs = np.zeros(len(msgs) + 1, dtype=np.uint64)
    if msgs:
        np.cumsum([len(m) for m in msgs], out=offs[1:])
    return b"".join(msgs), offs


class Engine:
    """Batched SPHINCS+ signing on one CUDA device."""

    def __init__(self, device: int | None = None):
        L = _lib.lib()
        self.device = _lib.default_device() if device is None else int(device)
        h = ctypes.c_void_p()
        rc = L.hs_open(self.device, ctypes.byref(h))
        if rc != _lib.HS_OK or not h.value:
            raise HeroSignError(f"hs_open(device={self.device}) failed (rc={rc}): no usable CUDA device")
        self._h = h
        # One handle is not reentrant (include/herosign_b200.h).  Every call
        # into the library holds this lock; callers that chain several calls
        # (upload keys -> override config -> sign -> restore, as sigcore does)
        # hold ``engine.lock`` across the whole sequence so another thread
        # cannot swap the key table or the config in between.
        self._lock = threading.RLock()
        self._keys: dict[str, bytes] = {}

    # -- lifecycle -------------------------------------------------------
    @property
    def lock(self) -> threading.RLock:
        """Re-entrant lock serialising this handle's calls (hold it across a
        multi-call sequence that must see one key table and config)."""
        return self._lock

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            with self._lock:
                _lib.lib().hs_close(self._h)
                self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int, what: str) -> None:
        _lib.check(self._h, rc, what)

    # -- device / config -------------------------------------------------
    def device_info(self) -> dict:
        v = [ctypes.c_int32() for _ in range(4)]
        self._check(_lib.lib().hs_device_info(self._h, *[ctypes.byref(x) for x in v]), "hs_device_info")
        return {"sm_count": v[0].value, "smem_optin": v[1].value, "cc": (v[2].value, v[3].value)}

    def config(self, set_id: str) -> dict:
        c = _lib.SetConfig()
        with self._lock:
            self._check(_lib.lib().hs_config_get(self._h, SET_INDEX[set_id], ctypes.byref(c)), "hs_config_get")
        return {
            "fors_trees_per_set": c.fors_trees_per_set,
            "fors_sets_fused": c.fors_sets_fused,
            "fors_relax": bool(c.fors_relax),
            "variant": {k: int(c.variant[i]) for i, k in enumerate(KERNELS)},
            "use_graph": bool(c.use_graph),
            "chunk": c.chunk,
            "wots_from_tree": bool(c.wots_from_tree),
            "streams": c.streams,
            "shared_layers": c.shared_layers,
            "shared_auto": bool(c.shared_auto),
            "fors_cta_levels": c.fors_cta_levels,
            "tree_split": int(c.tree_split),
            "overlap": int(c.overlap),
            "fors_small_batch": int(c.fors_small_batch),
            "tree_small_batch": int(c.tree_small_batch),
        }

    def set_config(self, set_id: str, **kw) -> dict:
        with self._lock:
            return self._set_config(set_id, **kw)

    def _set_config(self, set_id: str, **kw) -> dict:
        cur = self.config(set_id)
        variant = dict(cur["variant"])
        variant.update(kw.pop("variant", {}) or {})
        cur.update(kw)
        c = _lib.SetConfig()
        c.fors_trees_per_set = int(cur["fors_trees_per_set"])
        c.fors_sets_fused = int(cur["fors_sets_fused"])
        c.fors_relax = int(bool(cur["fors_relax"]))
        for i, k in enumerate(KERNELS):
            c.variant[i] = int(variant[k])
        c.use_graph = int(bool(cur["use_graph"]))
        c.chunk = int(cur["chunk"])
        c.wots_from_tree = int(bool(cur["wots_from_tree"]))
        c.streams = int(cur["streams"])
        c.shared_layers = int(cur["shared_layers"])
        c.shared_auto = int(bool(cur["shared_auto"]))
        c.fors_cta_levels = int(cur["fors_cta_levels"])
        c.tree_split = int(cur["tree_split"])
        c.overlap = int(cur["overlap"])
        c.fors_small_batch = int(cur["fors_small_batch"])
        c.tree_small_batch = int(cur["tree_small_batch"])
        self._check(_lib.lib().hs_config_set(self._h, SET_INDEX[set_id], ctypes.byref(c)), "hs_config_set")
        return self.config(set_id)

    @staticmethod
    def fors_smem_bytes(set_id: str, trees_per_set: int, sets_fused: int, relax: bool) -> int:
        return int(_lib.lib().hs_fors_smem_bytes(SET_INDEX[set_id], trees_per_set, sets_fused, int(relax)))

    # -- keys ------------------------------------------------------------
    def upload_keys(self, set_id: str, sks: bytes | Iterable[bytes]) -> int:
        p = derive(set_id)
        blob = sks if isinstance(sks, (bytes, bytearray)) else b"".join(sks)
        blob = bytes(blob)
        if not blob or len(blob) % p.sk_bytes:
            raise UsageError(f"key table must be a non-empty multiple of {p.sk_bytes} bytes")
        with self._lock:
            if self._keys.get(set_id) == blob:
                return len(blob) // p.sk_bytes
            self._keys.pop(set_id, None)
            self._check(_lib.lib().hs_keys_upload(self._h, p.index, _u8ptr(blob), len(blob) // p.sk_bytes),
                        "hs_keys_upload")
            self._keys[set_id] = blob
        return len(blob) // p.sk_bytes

    def keygen_batch(self, set_id: str, seeds: Sequence[bytes]) -> list[bytes]:
        p = derive(set_id)
        for s in seeds:
            if len(s) != 3 * p.n:
                raise UsageError(f"seed must be {3 * p.n} bytes, got {len(s)}")
        if not seeds:
            return []
        blob = b"".join(seeds)
        out = bytearray(len(seeds) * p.sk_bytes)
        with self._lock:
            self._check(_lib.lib().hs_keygen_batch(self._h, p.index, _u8ptr(blob), len(seeds), _u8ptr(out)),
                        "hs_keygen_batch")
        return [bytes(out[i * p.sk_bytes:(i + 1) * p.sk_bytes]) for i in range(len(seeds))]

    # -- signing ---------------------------------------------------------
    def sign_into(self, set_id: str, blob, offs: np.ndarray, count: int, out, key_idx: np.ndarray | None = None,
                  opt_rand=None, wots_steps=None) -> None:
        """Zero-copy batch sign: inputs/outputs are caller buffers (pinned ones avoid staging).
        ``wots_steps`` (a uint32 array of ``count``, or a pointer) receives each
        message's WOTS_Sign F steps -- the data-dependent term of the exact
        compression count (hs_sign_batch_ex)."""
        p = derive(set_id)
        offs = _offsets(offs, count)
        key_idx = _key_index(key_idx, count)
        if opt_rand is not None and not isinstance(opt_rand, int) and len(opt_rand) < count * p.n:
            raise UsageError(f"opt_rand must be {p.n} bytes per message")
        if isinstance(wots_steps, np.ndarray) and (wots_steps.dtype != np.uint32 or wots_steps.size < count
                                                    or not wots_steps.flags.c_contiguous):
            raise UsageError(f"wots_steps must be a contiguous uint32 array of {count}")
        with self._lock:
            self._sign_into_nolock(p, blob, offs, count, out, key_idx, opt_rand, wots_steps)

    def _sign_into_nolock(self, p, blob, offs, count, out, key_idx, opt_rand, wots_steps) -> None:
        # the C call (arguments already validated); the caller holds this handle's lock
        self._check(
            _lib.lib().hs_sign_batch_ex(self._h, p.index, _u8ptr(blob), _u8ptr(offs),
                                        _u8ptr(key_idx) if key_idx is not None else None, _u8ptr(opt_rand),
                                        count, _u8ptr(out), _u8ptr(wots_steps)),
            "hs_sign_batch_ex")

    def sign_batch(self, set_id: str, msgs: Sequence[bytes], key_idx: Sequence[int] | None = None,
                   opt_rand: Sequence[bytes] | bytes | None = None, counts: bool = False):
        """Sign a list of messages; with ``counts`` also return each message's
        WOTS_Sign F steps (``(sigs, steps)``)."""
        p = derive(set_id)
        count = len(msgs)
        with self._lock:
            if set_id not in self._keys:
                raise UsageError("no keys uploaded for this parameter set")
            if not count:
                return ([], []) if counts else []
            return self._sign_batch(p, set_id, msgs, count, key_idx, opt_rand, counts)

    def _sign_batch(self, p, set_id, msgs, count, key_idx, opt_rand, counts):
        blob, offs = pack_messages(msgs)
        kidx = None
        if key_idx is not None:
            kidx = np.ascontiguousarray(key_idx, dtype=np.uint32)
            if kidx.shape != (count,):
                raise UsageError("key_idx must hold one entry per message")
        orand = None
        if opt_rand is not None:
            if isinstance(opt_rand, (bytes, bytearray)):
                orand = opt_rand
            else:
                # a None entry means the reference default, PK.seed of the message's key (sigcore.py:162-163)
                ks = self._keys[set_id]
                kk = kidx if kidx is not None else np.zeros(count, dtype=np.uint32)
                orand = b"".join(o if o is not None else ks[int(kk[i]) * p.sk_bytes + 2 * p.n:
                                                          int(kk[i]) * p.sk_bytes + 3 * p.n]
                                 for i, o in enumerate(opt_rand))
            if len(orand) != count * p.n:
                raise UsageError(f"opt_rand must be {p.n} bytes per message")
            orand = bytes(orand)
        out = bytearray(count * p.sig_bytes)
        steps = np.zeros(count, dtype=np.uint32) if counts else None
        self.sign_into(set_id, blob, offs, count, out, kidx, orand, steps)
        sb = p.sig_bytes
        sigs = [bytes(out[i * sb:(i + 1) * sb]) for i in range(count)]
        return (sigs, [int(x) for x in steps]) if counts else sigs

    def verify_batch(self, set_id: str, pks: Sequence[bytes] | bytes, msgs: Sequence[bytes], sigs: Sequence[bytes],
                     key_idx: Sequence[int] | None = None) -> list[bool]:
        p = derive(set_id)
        count = len(msgs)
        if len(sigs) != count:
            raise UsageError("one signature per message required")
        if count == 0:
            return []
        pkb = pks if isinstance(pks, (bytes, bytearray)) else b"".join(pks)
        if not pkb or len(pkb) % p.pk_bytes:
            raise UsageError(f"public keys must be a multiple of {p.pk_bytes} bytes")
        ok = np.zeros(count, dtype=np.uint8)
        good = [len(s) == p.sig_bytes for s in sigs]
        sigblob = b"".join(s if g else bytes(p.sig_bytes) for s, g in zip(sigs, good))
        blob, offs = pack_messages(msgs)
        kidx = None if key_idx is None else np.ascontiguousarray(key_idx, dtype=np.uint32)
        with self._lock:
            self._verify_nolock(p, bytes(pkb), blob, offs, count, sigblob, kidx, ok)
        return [bool(o) and g for o, g in zip(ok.tolist(), good)]

    def _verify_nolock(self, p, pkb: bytes, blob, offs, count, sigs, kidx, ok) -> None:
        self._check(_lib.lib().hs_verify_batch(self._h, p.index, _u8ptr(pkb), len(pkb) // p.pk_bytes,
                                               _u8ptr(blob), _u8ptr(offs), _u8ptr(kidx), _u8ptr(sigs), count,
                                               _u8ptr(ok)),
                    "hs_verify_batch")

    def verify_into(self, set_id: str, pks: bytes, blob, offs: np.ndarray, count: int, sigs,
                    key_idx: np.ndarray | None = None) -> np.ndarray:
        """Zero-copy batch verify: messages as (blob, offs) and signatures as one
        buffer of count * sig_bytes (bytes, or a pointer such as the pinned buffer
        sign_into just filled).  Returns a bool array."""
        p = derive(set_id)
        if not pks or len(pks) % p.pk_bytes:
            raise UsageError(f"public keys must be a multiple of {p.pk_bytes} bytes")
        ok = np.zeros(count, dtype=np.uint8)
        offs = _offsets(offs, count)
        kidx = _key_index(key_idx, count)
        with self._lock:
            self._check(_lib.lib().hs_verify_batch(self._h, p.index, _u8ptr(bytes(pks)), len(pks) // p.pk_bytes,
                                                   _u8ptr(blob), _u8ptr(offs), _u8ptr(kidx), _u8ptr(sigs),
                                                   count, _u8ptr(ok)),
                        "hs_verify_batch")
        return ok.astype(bool)

    # -- device-resident stages (bench / graph signer) ---------------------
    def stage(self, set_id: str, blob, offs: np.ndarray, count: int, key_idx=None, opt_rand=None) -> None:
        p = derive(set_id)
        offs = _offsets(offs, count)
        key_idx = _key_index(key_idx, count)
        if opt_rand is not None and not isinstance(opt_rand, int) and len(opt_rand) < count * p.n:
            raise UsageError(f"opt_rand must be {p.n} bytes per message")
        with self._lock:
            self._check(_lib.lib().hs_stage(self._h, p.index, _u8ptr(blob), _u8ptr(offs), _u8ptr(key_idx),
                                            _u8ptr(opt_rand), count), "hs_stage")

    def run(self, set_id: str, count: int, mode: int = 0) -> None:
        with self._lock:
            self._check(_lib.lib().hs_run(self._h, SET_INDEX[set_id], count, mode), "hs_run")

    def sync(self) -> None:
        with self._lock:
            self._check(_lib.lib().hs_sync(self._h), "hs_sync")

    def fetch(self, set_id: str, first: int, count: int, out) -> None:
        with self._lock:
            self._check(_lib.lib().hs_fetch(self._h, SET_INDEX[set_id], first, count, _u8ptr(out)), "hs_fetch")

    def timings(self) -> dict:
        ms = (ctypes.c_float * 5)()
        with self._lock:
            n = _lib.lib().hs_timings(self._h, ms, 5)
        if n < 0:
            self._check(n, "hs_timings")
        names = ("batch", "msg_prep", "FORS_Sign", "TREE_Sign", "WOTS_Sign")
        return {names[i]: float(ms[i]) for i in range(max(n, 0))}

    def bench_run(self, set_id: str, count: int, steps: int, mode: int = 0, flush_bytes: int = 0) -> list[float]:
        """Per-step device ms of `steps` runs over the staged batch (CUDA events, launching stream)."""
        ms = (ctypes.c_float * steps)()
        with self._lock:
            self._check(
                _lib.lib().hs_bench_run(self._h, SET_INDEX[set_id], count, steps, mode, flush_bytes, ms),
                "hs_bench_run")
        return [float(x) for x in ms]

    def tune(self, set_id: str, count: int = 2048, top: int = 12, reps: int = 5) -> dict:
        """The native on-device Tree Tuning search (hs_tune): FORS layout,
        in-CTA levels, SHA-256 path per kernel and sub-batch streams, timed on
        this device; leaves the engine configured and returns the report."""
        import json

        cap = 1 << 16
        buf = ctypes.create_string_buffer(cap)
        with self._lock:
            rc = _lib.lib().hs_tune(self._h, SET_INDEX[set_id], int(count), int(top), int(reps), buf, cap)
        if rc < 0:
            self._check(rc, "hs_tune")
        if rc > 0:
            raise HeroSignError(f"hs_tune report needs {rc} bytes (config applied)")
        rep = json.loads(buf.value.decode())
        c = rep["config"]
        c["variant"] = dict(zip(KERNELS, c["variant"]))
        return rep

    @property
    def launch_count(self) -> int:
        return int(_lib.lib().hs_launch_count(self._h))

    def batch_info(self, set_id: str) -> dict:
        """How the staged batch runs: messages, subtree-sharing depth chosen by the
        auto policy, FORS levels kept in the CTA, split TREE_Sign, and the shared
        subtrees its last run computed."""
        v = (ctypes.c_int32 * 5)()
        with self._lock:
            n = _lib.lib().hs_batch_info(self._h, SET_INDEX[set_id], v, 5)
        if n < 0:
            self._check(n, "hs_batch_info")
        return {"staged": int(v[0]), "shared_layers": int(v[1]), "fors_cta_levels": int(v[2]),
                "tree_split": int(v[3]), "shared_subtrees_built": int(v[4])}

    def launch_stats(self, reset: bool = True) -> dict:
        """Host-side batch launch latency: cudaGraphLaunch calls since the last reset."""
        v = (ctypes.c_double * 3)()
        with self._lock:
            n = _lib.lib().hs_launch_stats(self._h, v, 3, 1 if reset else 0)
        if n < 0:
            self._check(n, "hs_launch_stats")
        return {"graph_launches": int(v[0]), "mean_us": float(v[1]), "max_us": float(v[2])}


class PinnedBuffer:
    """Page-locked host buffer (cudaMallocHost) exposed as a writable memoryview."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        ptr = _lib.lib().hs_host_alloc(max(self.nbytes, 1))
        if not ptr:
            raise HeroSignError(f"cudaMallocHost({nbytes}) failed")
        self.ptr = int(ptr)
        self.view = (ctypes.c_char * max(self.nbytes, 1)).from_address(self.ptr)

    def array(self, dtype=np.uint8) -> np.ndarray:
        return np.frombuffer(self.view, dtype=dtype)

    def free(self) -> None:
        if self.ptr:
            _lib.lib().hs_host_free(ctypes.c_void_p(self.ptr))
            self.ptr = 0

    def __del__(self):  # pragma: no cover
        try:
            self.free()
        except Exception:
            pass


def _addr(buf) -> int:
    """Address of a host buffer (bytes / bytearray / numpy array / raw pointer)."""
    ptr = _u8ptr(buf)
    return int(ptr or 0)


def shard_ranges(count: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous, balanced message ranges [first, first + n), one per device
    (messages are independent; no collective)."""
    if parts < 1:
        raise UsageError("at least one device is required")
    base, extra = divmod(count, parts)
    out, first = [], 0
    for g in range(parts):
        n = base + (1 if g < extra else 0)
        out.append((first, n))
        first += n
    return out


class _AllLocks:
    """Re-entrant lock over several engines' handle locks (taken in a fixed
    order), so a multi-call sequence owns every device's key table and config."""

    def __init__(self, locks):
        self._locks = list(locks)

    def acquire(self):
        for lk in self._locks:
            lk.acquire()
        return True

    def release(self):
        for lk in reversed(self._locks):
            lk.release()

    __enter__ = acquire

    def __exit__(self, *exc):
        self.release()


class MultiEngine:
    """Batched signing over several devices of one node.

    One ``Engine`` per entry of ``devices`` (a device may repeat: two handles on
    one device sign concurrently); a batch is split into contiguous balanced
    shards, each signed by its engine on its own host thread (ctypes releases
    the GIL around the C call) and copied by that engine straight into the
    caller's output at offset ``first * sig_bytes`` -- pinned outputs take the
    device's D2H directly.  No collective runs on the signing path; the only
    partition is by message, as the reference's m x T split
    (batchgraph.py:110-121) is.  Same calls as ``Engine`` for keys, config,
    signing and verification, so sigcore can drive it (``devices=``)."""

    def __init__(self, devices, engines: list | None = None):
        self.devices = [int(d) for d in devices]
        if not self.devices:
            raise UsageError("at least one device is required")
        if engines is None:
            engines, seen = [], set()
            for d in self.devices:
                if d in seen:  # another handle on a device already in use
                    e = Engine(d)
                    apply_tuned_config(e)
                else:
                    e = get_engine(d)
                    seen.add(d)
                engines.append(e)
        self.engines = list(engines)
        uniq = list({id(e): e for e in self.engines}.values())
        self.lock = _AllLocks(e.lock for e in uniq)

    def __len__(self) -> int:
        return len(self.engines)

    def upload_keys(self, set_id: str, sks) -> int:
        blob = bytes(sks if isinstance(sks, (bytes, bytearray)) else b"".join(sks))
        with self.lock:
            return [e.upload_keys(set_id, blob) for e in self.engines][0]

    def config(self, set_id: str) -> dict:
        return self.engines[0].config(set_id)

    def set_config(self, set_id: str, **kw) -> dict:
        with self.lock:
            return [e.set_config(set_id, **kw) for e in self.engines][0]

    @staticmethod
    def _parallel(jobs) -> None:
        errors: list = []

        def run(fn):
            try:
                fn()
            except Exception as exc:  # surfaced after join
                errors.append(exc)

        threads = [threading.Thread(target=run, args=(fn,)) for fn in jobs]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]

    def sign_into(self, set_id: str, blob, offs, count: int, out, key_idx=None, opt_rand=None,
                  wots_steps=None) -> None:
        """Engine.sign_into over all devices: shard g signs messages
        [first, first + n) into ``out`` at ``first * sig_bytes``."""
        p = derive(set_id)
        offs = _offsets(offs, count)
        key_idx = _key_index(key_idx, count)
        if opt_rand is not None and not isinstance(opt_rand, int) and len(opt_rand) < count * p.n:
            raise UsageError(f"opt_rand must be {p.n} bytes per message")
        if isinstance(wots_steps, np.ndarray) and (wots_steps.dtype != np.uint32 or wots_steps.size < count
                                                    or not wots_steps.flags.c_contiguous):
            raise UsageError(f"wots_steps must be a contiguous uint32 array of {count}")
        b_addr, o_addr = _addr(blob), _addr(out)
        r_addr = _addr(opt_rand) if opt_rand is not None else 0
        w_addr = _addr(wots_steps) if wots_steps is not None else 0
        jobs = []
        for eng, (first, n) in zip(self.engines, shard_ranges(count, len(self.engines))):
            if n == 0:
                continue
            o = np.ascontiguousarray(offs[first:first + n + 1])
            k = np.ascontiguousarray(key_idx[first:first + n]) if key_idx is not None else None
            jobs.append(lambda eng=eng, first=first, n=n, o=o, k=k: eng._sign_into_nolock(
                p, b_addr, o, n, o_addr + first * p.sig_bytes, k, r_addr + first * p.n if r_addr else None,
                w_addr + 4 * first if w_addr else None))
        with self.lock:  # the worker threads run under the caller's ownership of every handle
            self._parallel(jobs)

    def sign_batch(self, set_id: str, msgs, key_idx=None, opt_rand=None, counts: bool = False):
        """Engine.sign_batch over all devices (same arguments and result)."""
        p = derive(set_id)
        count = len(msgs)
        if not count:
            return ([], []) if counts else []
        blob, offs = pack_messages([bytes(m) for m in msgs])
        kidx = _key_index(key_idx, count)
        orand = None
        if opt_rand is not None:
            if isinstance(opt_rand, (bytes, bytearray)):
                orand = bytes(opt_rand)
            else:
                if any(o is None for o in opt_rand):
                    raise UsageError("resolve default opt_rand entries (PK.seed) before a multi-device sign")
                orand = b"".join(opt_rand)
            if len(orand) != count * p.n:
                raise UsageError(f"opt_rand must be {p.n} bytes per message")
        out = bytearray(count * p.sig_bytes)
        steps = np.zeros(count, dtype=np.uint32)
        self.sign_into(set_id, blob, offs, count, out, kidx, orand, steps)
        sb = p.sig_bytes
        sigs = [bytes(out[i * sb:(i + 1) * sb]) for i in range(count)]
        return (sigs, [int(x) for x in steps]) if counts else sigs

    def verify_batch(self, set_id: str, pks, msgs, sigs, key_idx=None) -> list[bool]:
        """Engine.verify_batch over all devices."""
        p = derive(set_id)
        count = len(msgs)
        if len(sigs) != count:
            raise UsageError("one signature per message required")
        if not count:
            return []
        pkb = bytes(pks if isinstance(pks, (bytes, bytearray)) else b"".join(pks))
        if not pkb or len(pkb) % p.pk_bytes:
            raise UsageError(f"public keys must be a multiple of {p.pk_bytes} bytes")
        good = [len(x) == p.sig_bytes for x in sigs]
        sigblob = b"".join(x if g else bytes(p.sig_bytes) for x, g in zip(sigs, good))
        blob, offs = pack_messages([bytes(m) for m in msgs])
        kidx = _key_index(key_idx, count)
        ok = np.zeros(count, dtype=np.uint8)
        b_addr, s_addr, ok_addr = _addr(blob), _addr(sigblob), _addr(ok)
        jobs = []
        for eng, (first, n) in zip(self.engines, shard_ranges(count, len(self.engines))):
            if n == 0:
                continue
            o = np.ascontiguousarray(offs[first:first + n + 1])
            k = np.ascontiguousarray(kidx[first:first + n]) if kidx is not None else None
            jobs.append(lambda eng=eng, first=first, n=n, o=o, k=k: eng._verify_nolock(
                p, pkb, b_addr, o, n, s_addr + first * p.sig_bytes, k, ok_addr + first))
        with self.lock:
            self._parallel(jobs)
        return [bool(x) and g for x, g in zip(ok.tolist(), good)]


_ENGINES: dict[int, Engine] = {}
_ENGINES_LOCK = threading.Lock()
_MULTI: dict[tuple, MultiEngine] = {}


TUNED_CONFIG = _lib.PKG_DIR / "b200_tuned.json"


def apply_tuned_config(eng: Engine, path=None) -> bool:
    """Apply $HERO_SIGN_CONFIG, else the packaged on-device tuning result
    (b200_tuned.json written by tools/tune_all.py on a B200), if present."""
    import os

    from .config import ENV_CONFIG_PATH, TuningConfig

    path = path or os.environ.get(ENV_CONFIG_PATH) or (TUNED_CONFIG if TUNED_CONFIG.exists() else None)
    if not path:
        return False
    TuningConfig.load(path).apply(eng)
    return True


def get_engine(device: int | None = None) -> Engine:
    """Process-wide engine for a device (default: $HEROSIGN_DEVICE / $LOCAL_RANK / 0),
    configured from the persisted tuning result when one exists."""
    dev = _lib.default_device() if device is None else int(device)
    with _ENGINES_LOCK:
        eng = _ENGINES.get(dev)
        if eng is None:
            eng = Engine(dev)
            apply_tuned_config(eng)
            _ENGINES[dev] = eng
        return eng


def get_multi_engine(devices) -> MultiEngine:
    """Process-wide MultiEngine for a device list (e.g. ``range(8)``), built on
    the per-device engines of ``get_engine``."""
    key = tuple(int(d) for d in devices)
    with _ENGINES_LOCK:
        m = _MULTI.get(key)
    if m is None:
        m = MultiEngine(key)
        with _ENGINES_LOCK:
            m = _MULTI.setdefault(key, m)
    return m
