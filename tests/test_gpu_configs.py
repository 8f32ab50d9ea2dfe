"""BASELINE.json configs 3-5 at their own sizes on the GPU, plus the on-device
Tree Tuning search (reference tuner.py:91-143, 222-274; sigcore.py:139-178).

* C3: 192f x 16,384 messages with the tuned configuration -- every signature
  verified on the GPU, 256 seeded ones byte-compared with the oracle.
* C4: 256f x 65,536 messages through hs_sign_batch into a pinned output
  (4 pipelined chunks of 16,384) -- every signature verified on the GPU, the
  first, last and a random message of each chunk byte-compared with the oracle.
* C5-mini: 2^16 messages over 1,024 keys (key_idx = i mod 1024, GPU keygen) --
  every signature verified on the GPU, one per key byte-compared with the oracle.
* Tree Tuning: the Python search (tuner.tune_on_device) and the native one
  (hs_tune) on 192f; the chosen layout is feasible and the tuned engine signs
  bit-exact.
"""

from __future__ import annotations

import random

import numpy as np
import pytest

import paper_2512_23969_b200 as hs
from paper_2512_23969_b200.engine import PinnedBuffer, pack_messages
from paper_2512_23969_b200.params import derive

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    return hs.get_engine()


def _sign_pinned(eng, set_id, msgs, key_idx=None):
    p = derive(set_id)
    blob, offs = pack_messages(msgs)
    out = PinnedBuffer(len(msgs) * p.sig_bytes)
    eng.sign_into(set_id, blob, offs, len(msgs), out.ptr, key_idx)
    return out, blob, offs


def _verify_all(eng, set_id, pks: bytes, blob, offs, count, out, key_idx=None) -> np.ndarray:
    return eng.verify_into(set_id, pks, blob, offs, count, out.ptr, key_idx)


def test_config3_192f_16384_tuned(eng, oracle_mod):
    set_id, count = "192f", 16384
    p = derive(set_id)
    rng = random.Random(2512_23969)
    sk = eng.keygen_batch(set_id, [rng.randbytes(3 * p.n)])[0]
    msgs = [rng.randbytes(32) for _ in range(count)]
    eng.upload_keys(set_id, sk)
    out, blob, offs = _sign_pinned(eng, set_id, msgs)
    try:
        ok = _verify_all(eng, set_id, sk[2 * p.n:], blob, offs, count, out)
        assert ok.all(), np.flatnonzero(~ok)[:10]
        pick = sorted(random.Random(3).sample(range(count), 256))
        ref, _ = oracle_mod.sign_many(set_id, sk, None, [msgs[i] for i in pick])
        raw = out.view
        bad = [i for i, r in zip(pick, ref) if raw[i * p.sig_bytes:(i + 1) * p.sig_bytes] != r]
        assert not bad, bad[:10]
    finally:
        out.free()


def test_config4_256f_65536_chunked(eng, oracle_mod):
    set_id, count = "256f", 65536
    p = derive(set_id)
    rng = random.Random(2512_23969)
    sk = eng.keygen_batch(set_id, [rng.randbytes(3 * p.n)])[0]
    msgs = [rng.randbytes(32) for _ in range(count)]
    eng.upload_keys(set_id, sk)
    chunk = eng.config(set_id)["chunk"]
    assert count // chunk >= 4  # several pipelined chunks per call
    out, blob, offs = _sign_pinned(eng, set_id, msgs)
    try:
        ok = _verify_all(eng, set_id, sk[2 * p.n:], blob, offs, count, out)
        assert ok.all(), np.flatnonzero(~ok)[:10]
        r = random.Random(4)
        pick = sorted({i for c0 in range(0, count, chunk)
                       for i in (c0, min(count, c0 + chunk) - 1, r.randrange(c0, min(count, c0 + chunk)))})
        ref, _ = oracle_mod.sign_many(set_id, sk, None, [msgs[i] for i in pick])
        raw = out.view
        bad = [i for i, x in zip(pick, ref) if raw[i * p.sig_bytes:(i + 1) * p.sig_bytes] != x]
        assert not bad, bad
    finally:
        out.free()


@pytest.mark.parametrize("set_id,count", [("128f", 1 << 16), ("192f", 1 << 14), ("256f", 1 << 13)])
def test_config5_mini_1024_keys(eng, oracle_mod, set_id, count):
    nkeys = 1024
    p = derive(set_id)
    rng = random.Random(1024 + p.n)
    sks = eng.keygen_batch(set_id, [rng.randbytes(3 * p.n) for _ in range(nkeys)])
    msgs = [rng.randbytes(32) for _ in range(count)]
    kidx = np.arange(count, dtype=np.uint32) % nkeys
    eng.upload_keys(set_id, sks)
    out, blob, offs = _sign_pinned(eng, set_id, msgs, kidx)
    try:
        pks = b"".join(k[2 * p.n:] for k in sks)
        ok = _verify_all(eng, set_id, pks, blob, offs, count, out, kidx)
        assert ok.all(), np.flatnonzero(~ok)[:10]
        r = random.Random(5)
        pick = [k + nkeys * r.randrange(count // nkeys) for k in range(nkeys)]  # one message of every key
        ref, _ = oracle_mod.sign_many(set_id, b"".join(sks), [int(kidx[i]) for i in pick], [msgs[i] for i in pick])
        raw = out.view
        bad = [i for i, x in zip(pick, ref) if raw[i * p.sig_bytes:(i + 1) * p.sig_bytes] != x]
        assert not bad, bad[:10]
    finally:
        out.free()


def _tuned_signs_exact(eng, oracle_mod, set_id):
    p = derive(set_id)
    rng = random.Random(8)
    sk = oracle_mod.keygen(set_id, rng.randbytes(3 * p.n))
    msgs = [rng.randbytes(rng.choice([0, 32, 100])) for _ in range(300)]
    eng.upload_keys(set_id, sk)
    sigs = eng.sign_batch(set_id, msgs)
    ref, _ = oracle_mod.sign_many(set_id, sk, None, msgs)
    assert sigs == ref


@pytest.mark.parametrize("native", [False, True])
def test_on_device_tree_tuning(eng, oracle_mod, native):
    from paper_2512_23969_b200.tuner import device_candidates, tune_on_device

    set_id = "192f"
    p = derive(set_id)
    base = eng.config(set_id)
    try:
        if native:
            rep = eng.tune(set_id, count=512, top=3, reps=1)
            assert rep["candidates"] == len(device_candidates(p, eng.device_info()["smem_optin"], alpha=0.0))
            best = min(rep["layouts"], key=lambda r: r["fors_ms"])
            layout = (best["trees_per_set"], best["sets_fused"], bool(best["relax"]))
        else:
            rep = tune_on_device(eng, set_id, count=512, top=3, reps=1)
            b = rep["best_layout"]
            layout = (b["trees_per_set"], b["sets_fused"], bool(b["relax"]))
        cfg = eng.config(set_id)
        assert (cfg["fors_trees_per_set"], cfg["fors_sets_fused"], cfg["fors_relax"]) == layout
        # step 4: the batch-size rules were timed (graph device times) and set
        assert "overlap_ms" in rep and "small_batch_ms" in rep
        assert cfg["fors_small_batch"] in (0, 16, 64, 256) and cfg["tree_small_batch"] in (0, 16, 64, 256)
        assert cfg["overlap"] >= 0 and "tree_small_batch_ms" in rep
        lanes = layout[0] * (p.fors_t // 2 if layout[2] else p.fors_t)
        assert lanes <= 768 and layout[0] * layout[1] <= p.k
        assert hs.Engine.fors_smem_bytes(set_id, *layout) <= eng.device_info()["smem_optin"]
        _tuned_signs_exact(eng, oracle_mod, set_id)
    finally:
        eng.set_config(set_id, **base)
