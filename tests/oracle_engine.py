"""CPU stand-in for ``Engine`` in host-side tests (no GPU in the build container).

It answers the calls ``sigcore.sign_on_engine`` makes -- ``lock``,
``upload_keys``, ``config`` / ``set_config``, ``sign_batch(..., counts=True)``
-- with bytes from the oracle (oracle/hs_oracle.c), so the host logic around
the engine (GraphSigner, the reference's scheduler, ctx_out accounting) can be
exercised on CPU.  Test infrastructure only: the package itself never imports
the oracle and has no CPU signing path.
"""

from __future__ import annotations

import threading

from paper_2512_23969_b200.params import compressions_per_signature, derive


def oracle_wots_steps(oracle, set_id: str, sk: bytes, msg: bytes, opt_rand: bytes | None = None) -> int:
    """WOTS_Sign F steps of one signature (sum of the signed base-w digits over
    all d layers), from the oracle's compression counter.  The oracle's count is
    the reference's sign_oracle path, which re-derives each of the k selected
    FORS secrets once more than the default path (SURVEY.md Appendix C,
    oracle.py:136-138 vs vexec.py:404-426); tests/test_host.py pins the relation
    against the reference's own counts."""
    p = derive(set_id)
    sigs, comps = oracle.sign_many(set_id, sk, None, [msg], opt_rand)
    fixed = compressions_per_signature(p, len(msg), digit_sum=0)["total"]
    return int(comps - p.k - fixed)


class OracleEngine:
    def __init__(self, oracle):
        self.oracle = oracle
        self.lock = threading.RLock()
        self._keys: dict[str, list[bytes]] = {}
        self._cfg: dict[str, dict] = {}
        self.sign_calls = 0

    def upload_keys(self, set_id, sks):
        blob = sks if isinstance(sks, (bytes, bytearray)) else b"".join(sks)
        p = derive(set_id)
        self._keys[set_id] = [bytes(blob[i:i + p.sk_bytes]) for i in range(0, len(blob), p.sk_bytes)]
        return len(self._keys[set_id])

    def config(self, set_id):
        return dict(self._cfg.get(set_id, {"fors_trees_per_set": 1, "fors_sets_fused": 1, "fors_relax": False,
                                           "variant": {"FORS_Sign": 0, "TREE_Sign": 0, "WOTS_Sign": 0, "host": 0}}))

    def set_config(self, set_id, **kw):
        c = self.config(set_id)
        c.update(kw)
        self._cfg[set_id] = c
        return c

    def sign_batch(self, set_id, msgs, key_idx=None, opt_rand=None, counts=False):
        self.sign_calls += 1
        keys = self._keys[set_id]
        kk = list(key_idx) if key_idx is not None else [0] * len(msgs)
        orand = list(opt_rand) if opt_rand is not None else [None] * len(msgs)
        sigs = [self.oracle.sign(set_id, keys[k], m, o) for m, k, o in zip(msgs, kk, orand)]
        if not counts:
            return sigs
        steps = [oracle_wots_steps(self.oracle, set_id, keys[k], m, o) for m, k, o in zip(msgs, kk, orand)]
        return sigs, steps


class OracleHandle(OracleEngine):
    """Per-device handle stand-in for ``MultiEngine`` on CPU: implements the raw
    pointer-level shard call (``_sign_into_nolock``) by reading the caller's
    buffers at the given addresses and writing the oracle's signatures and WOTS
    step counts back at the shard's offsets -- so the sharding and offset
    arithmetic of MultiEngine runs unchanged."""

    def __init__(self, oracle, device: int = 0):
        super().__init__(oracle)
        self.device = device
        self.shards: list[tuple[int, int]] = []  # (messages, output address) per call

    def _sign_into_nolock(self, p, blob, offs, count, out, key_idx, opt_rand, wots_steps):
        import ctypes

        import numpy as np

        keys = self._keys[p.id]
        base = int(blob)
        msgs = [ctypes.string_at(base + int(offs[i]), int(offs[i + 1] - offs[i])) for i in range(count)]
        kk = [int(x) for x in key_idx] if key_idx is not None else [0] * count
        self.shards.append((count, int(out)))
        for i, (m, k) in enumerate(zip(msgs, kk)):
            o = ctypes.string_at(int(opt_rand) + i * p.n, p.n) if opt_rand else None
            sig = self.oracle.sign(p.id, keys[k], m, o)
            ctypes.memmove(int(out) + i * p.sig_bytes, sig, p.sig_bytes)
            if wots_steps:
                v = np.array([oracle_wots_steps(self.oracle, p.id, keys[k], m, o)], dtype=np.uint32)
                ctypes.memmove(int(wots_steps) + 4 * i, v.ctypes.data, 4)
