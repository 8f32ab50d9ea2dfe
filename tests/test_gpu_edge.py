"""GPU edge cases: long and empty messages, extreme seeds, single-message and
odd-sized batches, repeated batches through a captured graph."""

from __future__ import annotations

import random

import numpy as np
import pytest

from conftest import SETS

import paper_2512_23969_b200 as hs
from paper_2512_23969_b200.params import compressions_per_signature, derive

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    return hs.get_engine()


@pytest.mark.parametrize("set_id", SETS)
def test_long_and_empty_messages(eng, oracle_mod, set_id):
    p = derive(set_id)
    rng = random.Random(3)
    sk = oracle_mod.keygen(set_id, rng.randbytes(3 * p.n))
    msgs = [b"", rng.randbytes(5000), b"\x00", rng.randbytes(70001), rng.randbytes(64 * 7 - 9)]
    eng.upload_keys(set_id, sk)
    sigs = eng.sign_batch(set_id, msgs)
    for m, s in zip(msgs, sigs):
        assert s == oracle_mod.sign(set_id, sk, m)
    assert all(eng.verify_batch(set_id, sk[2 * p.n:], msgs, sigs))


@pytest.mark.parametrize("set_id", SETS)
def test_extreme_seeds(eng, oracle_mod, set_id):
    p = derive(set_id)
    seeds = [bytes(3 * p.n), b"\xff" * (3 * p.n)]
    sks = eng.keygen_batch(set_id, seeds)
    assert sks == [oracle_mod.keygen(set_id, s) for s in seeds]
    eng.upload_keys(set_id, sks)
    msgs = [b"\xff" * 33, bytes(32)]
    sigs = eng.sign_batch(set_id, msgs, key_idx=[1, 0], opt_rand=[b"\xff" * p.n, bytes(p.n)])
    assert sigs[0] == oracle_mod.sign(set_id, sks[1], msgs[0], b"\xff" * p.n)
    assert sigs[1] == oracle_mod.sign(set_id, sks[0], msgs[1], bytes(p.n))


@pytest.mark.parametrize("count", [1, 7, 257, 1031])
def test_batch_sizes_and_graph_replay(eng, oracle_mod, count):
    """Odd batch sizes (partial warps / blocks / sub-batches); the same shape twice
    replays the captured graph and must give the same bytes."""
    p = derive("128f")
    rng = random.Random(count)
    sk = oracle_mod.keygen("128f", rng.randbytes(48))
    msgs = [rng.randbytes(32) for _ in range(count)]
    eng.upload_keys("128f", sk)
    first = eng.sign_batch("128f", msgs)
    again = eng.sign_batch("128f", msgs)
    assert first == again
    check = sorted({0, count - 1, count // 2})
    ref, _ = oracle_mod.sign_many("128f", sk, None, [msgs[i] for i in check])
    assert [first[i] for i in check] == ref
    assert all(eng.verify_batch("128f", sk[32:], msgs, first))


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("set_id", SETS)
def test_chunked_multistream_mixed_keys(eng, oracle_mod, set_id, overlap):
    """hs_sign_batch over several chunks (chunk < count), 4 weighted sub-batches
    per chunk (FORS || TREE streams and concurrent sub-batches, or one stream
    order), two keys, mixed opt_rand: every signature equals the oracle's."""
    p = derive(set_id)
    rng = random.Random(4242 + p.n)
    sks = [oracle_mod.keygen(set_id, rng.randbytes(3 * p.n)) for _ in range(2)]
    count = 2600 if set_id == "128f" else 1100
    msgs = [rng.randbytes(rng.choice([0, 32, 100])) for _ in range(count)]
    kidx = [rng.randrange(2) for _ in range(count)]
    opts = [rng.randbytes(p.n) if i % 5 == 0 else None for i in range(count)]
    eng.upload_keys(set_id, sks)
    base = eng.config(set_id)
    try:
        eng.set_config(set_id, chunk=1024, streams=4, overlap=overlap)
        sigs, steps = eng.sign_batch(set_id, msgs, key_idx=kidx, opt_rand=opts, counts=True)
    finally:
        eng.set_config(set_id, **base)
    # oracle: opt_rand None means PK.seed (sigcore.py:162-163)
    blob = b"".join(o if o is not None else sks[k][2 * p.n:3 * p.n] for o, k in zip(opts, kidx))
    ref, comps = oracle_mod.sign_many(set_id, b"".join(sks), kidx, msgs, blob)
    bad = [i for i in range(count) if sigs[i] != ref[i]]
    assert not bad, bad[:10]
    # the per-message WOTS step counts add up to the oracle's compression count
    # (oracle path = default path + k re-derived FORS secrets, tests/oracle_engine.py)
    fixed = sum(compressions_per_signature(p, len(m), digit_sum=0)["total"] for m in msgs)
    assert sum(steps) == comps - count * p.k - fixed
    assert all(0 <= x <= p.d * p.wots_len * (p.w - 1) for x in steps)


@pytest.mark.parametrize("pinned", [False, True])
def test_pipelined_chunks_io(eng, oracle_mod, pinned):
    """hs_sign_batch_ex's two-slot pipeline over 4 chunks (the last one ragged),
    with pinned or pageable message / signature / step-count buffers: the bytes
    and counts equal a single-chunk run, and sampled signatures the oracle's."""
    from paper_2512_23969_b200.engine import PinnedBuffer, pack_messages

    set_id = "192f"
    p = derive(set_id)
    rng = random.Random(99)
    sks = [oracle_mod.keygen(set_id, rng.randbytes(3 * p.n)) for _ in range(3)]
    count = 1000
    msgs = [rng.randbytes(rng.choice([1, 32, 90])) for _ in range(count)]
    kidx = np.array([rng.randrange(3) for _ in range(count)], dtype=np.uint32)
    eng.upload_keys(set_id, sks)
    blob, offs = pack_messages(msgs)
    base = eng.config(set_id)
    bufs = []
    try:
        eng.set_config(set_id, chunk=count)
        one, one_steps = eng.sign_batch(set_id, msgs, key_idx=kidx, counts=True)
        eng.set_config(set_id, chunk=300, streams=3)
        if pinned:
            mb, ob, sb = PinnedBuffer(len(blob)), PinnedBuffer(count * p.sig_bytes), PinnedBuffer(4 * count)
            bufs = [mb, ob, sb]
            mb.array()[:] = np.frombuffer(blob, dtype=np.uint8)
            eng.sign_into(set_id, mb.ptr, offs, count, ob.ptr, kidx, None, sb.ptr)
            raw, steps = bytes(ob.view), [int(x) for x in sb.array(np.uint32)]
        else:
            out, st = bytearray(count * p.sig_bytes), np.zeros(count, dtype=np.uint32)
            eng.sign_into(set_id, blob, offs, count, out, kidx, None, st)
            raw, steps = bytes(out), [int(x) for x in st]
    finally:
        eng.set_config(set_id, **base)
        for b in bufs:
            b.free()
    sigs = [raw[i * p.sig_bytes:(i + 1) * p.sig_bytes] for i in range(count)]
    assert sigs == one and steps == one_steps
    check = [0, 299, 300, 599, 600, 899, 900, 999]
    ref, _ = oracle_mod.sign_many(set_id, b"".join(sks), [int(kidx[i]) for i in check], [msgs[i] for i in check])
    assert [sigs[i] for i in check] == ref


def test_verify_into_pinned_roundtrip(eng, oracle_mod):
    """verify_into reads the pinned buffer sign_into filled; a flipped byte fails only its message."""
    import numpy as np

    from paper_2512_23969_b200.engine import PinnedBuffer, pack_messages

    set_id = "128f"
    p = derive(set_id)
    rng = random.Random(808)
    sk = oracle_mod.keygen(set_id, rng.randbytes(3 * p.n))
    eng.upload_keys(set_id, sk)
    msgs = [rng.randbytes(rng.choice([0, 32, 90])) for _ in range(300)]
    blob, offs = pack_messages(msgs)
    out = PinnedBuffer(len(msgs) * p.sig_bytes)
    try:
        eng.sign_into(set_id, blob, offs, len(msgs), out.ptr)
        assert eng.verify_into(set_id, sk[2 * p.n:], blob, offs, len(msgs), out.ptr).all()
        out.array()[17 * p.sig_bytes + 1234] ^= 0x40
        ok = eng.verify_into(set_id, sk[2 * p.n:], blob, offs, len(msgs), out.ptr)
        assert not ok[17] and ok.sum() == len(msgs) - 1
        raw = bytes(out.view[: 3 * p.sig_bytes])
        assert raw[:p.sig_bytes] == oracle_mod.sign(set_id, sk, msgs[0])
    finally:
        out.free()


def test_reference_call_knobs(eng, oracle_mod):
    """sigcore.sign's per-call fusion / relax / selection knobs (sigcore.py:139-153)
    change only the execution shape: same bytes, engine config restored."""

    class Selection:  # duck-typed reference BackendSelection (backends.py:201-257)
        def __init__(self, v):
            self.v = v

        def get(self, kernel, set_id):
            return self.v

    set_id = "192f"
    p = derive(set_id)
    seed = random.Random(55).randbytes(3 * p.n)
    sk = hs.keygen(set_id, seed)
    msg = b"per-call knobs"
    ref = oracle_mod.sign(set_id, sk.to_bytes(), msg)
    base = eng.config(set_id)
    for sel in (Selection("baseline"), Selection("tuned")):
        assert hs.sign(msg, sk, set_id, selection=sel) == ref
    fusion = type("Fusion", (), {"trees_per_set": 2, "sets_fused": 3})()
    assert hs.sign(msg, sk, set_id, fusion=fusion, relax=True) == ref
    assert hs.get_engine().config(set_id) == base


def test_multi_engine_two_handles_one_device(eng, oracle_mod):
    """MultiEngine with two handles on device 0 (the multi-GPU path on a
    one-GPU box): contiguous shards signed concurrently into one pinned output
    at the right offsets, bit-exact vs the oracle, exact step counts; and the
    public sign_batch / verify_batch with devices=[0, 0]."""
    from paper_2512_23969_b200.engine import Engine, MultiEngine, PinnedBuffer, pack_messages

    set_id = "128f"
    p = derive(set_id)
    rng = random.Random(77)
    sks = [oracle_mod.keygen(set_id, rng.randbytes(3 * p.n)) for _ in range(2)]
    count = 777
    msgs = [rng.randbytes(rng.choice([0, 32, 64, 65, 200])) for _ in range(count)]
    kidx = np.array([rng.randrange(2) for _ in range(count)], dtype=np.uint32)
    second = Engine(0)
    out = PinnedBuffer(count * p.sig_bytes)
    try:
        multi = MultiEngine([0, 0], engines=[eng, second])
        multi.upload_keys(set_id, sks)
        blob, offs = pack_messages(msgs)
        steps = np.zeros(count, dtype=np.uint32)
        multi.sign_into(set_id, blob, offs, count, out.ptr, kidx, None, steps)
        raw = bytes(out.view)
    finally:
        out.free()
        second.close()
    sigs = [raw[i * p.sig_bytes:(i + 1) * p.sig_bytes] for i in range(count)]
    ref, comps = oracle_mod.sign_many(set_id, b"".join(sks), [int(k) for k in kidx], msgs)
    bad = [i for i in range(count) if sigs[i] != ref[i]]
    assert not bad, bad[:10]
    fixed = sum(compressions_per_signature(p, len(m), digit_sum=0)["total"] for m in msgs)
    assert int(steps.sum()) == comps - count * p.k - fixed

    keys = [hs.SecretKey.from_bytes(k, p) for k in sks]
    sub = list(range(0, count, 13))
    got = hs.sign_batch([msgs[i] for i in sub], keys, p, key_idx=[int(kidx[i]) for i in sub], devices=[0, 0])
    assert got == [ref[i] for i in sub]
    assert all(hs.verify_batch([msgs[i] for i in sub], got, [k.public() for k in keys], p,
                               key_idx=[int(kidx[i]) for i in sub], devices=[0, 0]))


def test_concurrent_public_calls_different_keys(eng, oracle_mod):
    """The reference's sign() is a pure function that callers use from many
    threads (sigcore.py:139-178).  Six threads share the process-wide engine,
    each with its own key and its own per-call FORS layout / SHA-path
    overrides, interleaving sign_batch and sign: every signature must be the
    oracle's under the caller's key, and the engine's configuration must come
    back unchanged (the key upload, overrides, sign and restore form one
    critical section, engine.Engine.lock)."""
    import threading

    set_id = "128f"
    p = derive(set_id)
    rng = random.Random(2024)
    keys = [hs.keygen(set_id, rng.randbytes(3 * p.n)) for _ in range(6)]
    work = [[rng.randbytes(rng.choice([0, 31, 32, 100])) for _ in range(9)] for _ in keys]
    fusions = [None, type("F", (), {"trees_per_set": 3, "sets_fused": 1})(), None,
               type("F", (), {"trees_per_set": 1, "sets_fused": 11})(), None, None]

    class Sel:  # duck-typed reference BackendSelection (backends.py:201-257)
        def __init__(self, v):
            self.v = v

        def get(self, kernel, set_id):
            return self.v

    sels = [None, None, Sel("baseline"), None, Sel("tuned"), None]
    base = eng.config(set_id)
    got: dict = {}
    errors: list = []
    start = threading.Barrier(len(keys))

    def worker(t):
        try:
            start.wait()
            out = []
            for r in range(3):
                if r == 1:
                    out += [hs.sign(m, keys[t], set_id, fusion=fusions[t], selection=sels[t]) for m in work[t][:3]]
                else:
                    out += hs.sign_batch(work[t], keys[t], set_id, fusion=fusions[t], selection=sels[t])
            got[t] = out
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(len(keys))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for t, k in enumerate(keys):
        ref = [oracle_mod.sign(set_id, k.to_bytes(), m) for m in work[t]]
        assert got[t] == ref + ref[:3] + ref, f"thread {t}"
    assert eng.config(set_id) == base


@pytest.mark.parametrize("set_id", SETS)
def test_chunks_with_small_tail_graph(eng, oracle_mod, set_id):
    """A call whose last chunk is a small graph: the full chunks run the
    throughput shape (tuned FORS layout, Merkle grid, the set's overlap rule)
    and the 3-message tail runs the small-graph shape (one FORS tree per CTA
    where enabled, warp-shuffle Merkle) inside the same pipelined call; every
    signature equals the oracle's and the step counts are exact."""
    p = derive(set_id)
    rng = random.Random(7070 + p.n)
    sk = oracle_mod.keygen(set_id, rng.randbytes(3 * p.n))
    count = 2 * 512 + 3
    msgs = [rng.randbytes(rng.choice([0, 32, 77])) for _ in range(count)]
    eng.upload_keys(set_id, sk)
    base = eng.config(set_id)
    try:
        eng.set_config(set_id, chunk=512)
        sigs, steps = eng.sign_batch(set_id, msgs, counts=True)
    finally:
        eng.set_config(set_id, **base)
    ref, comps = oracle_mod.sign_many(set_id, sk, None, msgs)
    bad = [i for i in range(count) if sigs[i] != ref[i]]
    assert not bad, bad[:10]
    fixed = sum(compressions_per_signature(p, len(m), digit_sum=0)["total"] for m in msgs)
    assert sum(steps) == comps - count * p.k - fixed
