"""GPU parity: the CUDA engine (through the C-ABI) against the reference's
golden fixtures and the C oracle.  Bit-exact: every signature byte must match."""

from __future__ import annotations

import hashlib
import random

import pytest

from conftest import GOLDEN_DIR, SETS

import paper_2512_23969_b200 as hs
from paper_2512_23969_b200.engine import variants
from paper_2512_23969_b200.params import derive

pytestmark = pytest.mark.gpu
H = bytes.fromhex


@pytest.fixture(scope="module")
def eng():
    return hs.get_engine()


@pytest.mark.parametrize("set_id", SETS)
def test_keygen_golden(eng, golden, set_id):
    g = golden["sets"][set_id]["keygen"]
    assert eng.keygen_batch(set_id, [H(g["seed"])])[0].hex() == g["sk"]
    sk = hs.keygen(set_id, H(g["seed"]))
    assert sk.to_bytes().hex() == g["sk"]


@pytest.mark.parametrize("set_id", SETS)
def test_sign_golden(eng, golden, set_id):
    g = golden["sets"][set_id]
    p = derive(set_id)
    for case in g["sign"]:
        sk = hs.SecretKey.from_bytes(H(case["sk"]), p)
        opt = H(case["opt_rand"]) if case["opt_rand"] else None
        ctx = []
        sig = hs.sign(H(case["msg"]), sk, p, opt_rand=opt, ctx_out=ctx)
        # ctx_out carries the reference's exact HashContext count (sigcore.py:166-168)
        assert ctx[0].compressions == case["compressions"], case["tag"]
        if case["tag"] == "zero":
            ref = (GOLDEN_DIR / f"sig_{set_id}_zero.bin").read_bytes()
            if sig != ref:
                bad = [i for i in range(len(ref)) if sig[i] != ref[i]]
                regions = hs.signature_regions(p)
                where = sorted({name for name, (lo, hi) in regions.items() for b in bad[:200] if lo <= b < hi})
                pytest.fail(f"{len(bad)} bytes differ; first at {bad[0]}; regions {where[:8]}")
        assert hashlib.sha256(sig).hexdigest() == case["sig_sha256"], case["tag"]


@pytest.mark.parametrize("set_id", SETS)
def test_bench_recipe_golden(eng, golden, set_id):
    g = golden["sets"][set_id]["bench_recipe"]
    rng = random.Random(2512_23969)
    p = derive(set_id)
    rng.randbytes(3 * p.n)
    msgs = [rng.randbytes(32) for _ in range(len(g["sig_sha256"]))]
    sigs = hs.sign_batch(msgs, hs.SecretKey.from_bytes(H(g["sk"]), p), p)
    assert [hashlib.sha256(s).hexdigest() for s in sigs] == g["sig_sha256"]


@pytest.mark.parametrize("set_id", SETS)
def test_mixed_batch_vs_oracle(eng, oracle_mod, set_id):
    """Ragged messages (0..300 B), several keys, explicit and default opt_rand."""
    p = derive(set_id)
    rng = random.Random(7 + p.n)
    seeds = [rng.randbytes(3 * p.n) for _ in range(3)]
    sks = [oracle_mod.keygen(set_id, s) for s in seeds]
    count = 40
    msgs = [rng.randbytes(rng.choice([0, 1, 3, 31, 32, 33, 55, 56, 64, 65, 119, 300])) for _ in range(count)]
    kidx = [rng.randrange(3) for _ in range(count)]
    opts = [rng.randbytes(p.n) if i % 3 == 0 else None for i in range(count)]
    keys = [hs.SecretKey.from_bytes(s, p) for s in sks]
    sigs = hs.sign_batch(msgs, keys, p, key_idx=kidx, opt_rand=opts)
    for i in range(count):
        ref = oracle_mod.sign(set_id, sks[kidx[i]], msgs[i], opts[i])
        assert sigs[i] == ref, i


@pytest.mark.parametrize("set_id", SETS)
@pytest.mark.parametrize("variant", range(len(variants())))
@pytest.mark.parametrize("stash", [True, False])
def test_layouts_and_variants(eng, oracle_mod, set_id, variant, stash):
    """Every FORS fusion layout / relax mode, every compiled SHA-256 path and both
    TREE_Sign shapes (split / fused) give identical bytes."""
    p = derive(set_id)
    rng = random.Random(99)
    seed = rng.randbytes(3 * p.n)
    sk = oracle_mod.keygen(set_id, seed)
    msgs = [rng.randbytes(32) for _ in range(6)]
    ref = [oracle_mod.sign(set_id, sk, m) for m in msgs]
    eng.upload_keys(set_id, sk)
    base = eng.config(set_id)
    # (N_tree, F, Relax); for 192f / 256f they cover both FORS_Sign
    # instantiations: the narrow 64-register kernel (<= 256 / 512 lanes: 192f
    # (1,1,0), (2,5,1); 256f (1,1,0), (2,2,1), (1,5,1)) and the 768-lane one
    layouts = {"128f": [(1, 1, 0), (11, 3, 0), (2, 5, 1), (16, 2, 1)],
               "192f": [(1, 1, 0), (3, 3, 0), (4, 2, 1), (2, 5, 1)],
               "256f": [(1, 1, 0), (2, 2, 1), (1, 5, 1), (3, 6, 1)]}[set_id]
    try:
        for i, (nt, f, rx) in enumerate(layouts):
            # cycle the TREE_Sign shapes: chain + leaf + Merkle grids, fused,
            # chain + leaf grid with warp-shuffle Merkle
            split = (2, 0, 1, 2)[i]
            eng.set_config(set_id, fors_trees_per_set=nt, fors_sets_fused=f, fors_relax=bool(rx), wots_from_tree=stash,
                           variant={k: variant for k in ("FORS_Sign", "TREE_Sign", "WOTS_Sign", "host")},
                           tree_split=split, fors_small_batch=0, tree_small_batch=0)  # run the shape as given
            assert eng.sign_batch(set_id, msgs) == ref, (nt, f, rx, split)
        assert eng.keygen_batch(set_id, [seed])[0] == sk  # keygen root kernel on this path
    finally:
        eng.set_config(set_id, **base)


@pytest.mark.parametrize("set_id", SETS)
def test_fors_upper_levels_split(eng, oracle_mod, set_id):
    """Any split between in-CTA FORS levels and the batch-wide level grids
    (fors_cta_levels -1 = auto, 0..log_t) gives identical bytes, with and
    without Relax and with uneven passes (vexec.py:437-463 semantics)."""
    p = derive(set_id)
    rng = random.Random(1234)
    sk = oracle_mod.keygen(set_id, rng.randbytes(3 * p.n))
    msgs = [rng.randbytes(rng.choice([0, 32, 77])) for _ in range(300)]
    ref, _ = oracle_mod.sign_many(set_id, sk, None, msgs)
    eng.upload_keys(set_id, sk)
    base = eng.config(set_id)
    try:
        for nt, f, rx in ((1, 1, 0), (1, 3, 0), (1, 2, 1), (base["fors_trees_per_set"], base["fors_sets_fused"],
                                                           int(base["fors_relax"]))):
            for lc in sorted({-1, 0, 1, 2, p.log_t - 1, p.log_t}):
                eng.set_config(set_id, fors_trees_per_set=nt, fors_sets_fused=f, fors_relax=bool(rx),
                               fors_cta_levels=lc, fors_small_batch=0)
                assert eng.sign_batch(set_id, msgs) == ref, (nt, f, rx, lc)
    finally:
        eng.set_config(set_id, **base)


def test_config_change_rebuilds_graph(eng, oracle_mod):
    """A captured batch graph is reused only for an identical config: toggling
    tree_split / fors_cta_levels on the same layout changes the kernels run."""
    set_id = "128f"
    p = derive(set_id)
    rng = random.Random(77)
    sk = oracle_mod.keygen(set_id, rng.randbytes(3 * p.n))
    msgs = [rng.randbytes(32) for _ in range(300)]
    ref, _ = oracle_mod.sign_many(set_id, sk, None, msgs)
    eng.upload_keys(set_id, sk)
    base = eng.config(set_id)
    try:
        counts = {}
        for split, lc in ((1, -1), (0, p.log_t), (1, -1), (2, -1)):
            eng.set_config(set_id, tree_split=split, fors_cta_levels=lc, streams=1, shared_layers=0,
                           tree_small_batch=0)
            n0 = eng.launch_count
            assert eng.sign_batch(set_id, msgs) == ref, (split, lc)
            counts.setdefault((split, lc), []).append(eng.launch_count - n0)
        # split TREE_Sign adds the leaf grid (and with 2 the Merkle grid);
        # leaves-only FORS adds log_t level grids
        assert counts[(1, -1)][0] - counts[(0, p.log_t)][0] == 1 + p.log_t
        assert counts[(2, -1)][0] - counts[(1, -1)][0] == 1
        assert counts[(1, -1)][0] == counts[(1, -1)][1]
    finally:
        eng.set_config(set_id, **base)


@pytest.mark.parametrize("set_id", SETS)
def test_verify_gpu(eng, golden, set_id):
    p = derive(set_id)
    g = golden["sets"][set_id]
    sk = H(g["keygen"]["sk"])
    pk = hs.PublicKey.from_bytes(sk[2 * p.n:], p)
    sig = (GOLDEN_DIR / f"sig_{set_id}_zero.bin").read_bytes()
    assert hs.verify(bytes(32), sig, pk, p)
    assert not hs.verify(bytes(31) + b"\x01", sig, pk, p)
    assert not hs.verify(bytes(32), sig[:-1], pk, p)
    rng = random.Random(5)
    bad = []
    for _ in range(24):
        b = bytearray(sig)
        b[rng.randrange(len(b))] ^= 1 << rng.randrange(8)
        bad.append(bytes(b))
    res = hs.verify_batch([bytes(32)] * len(bad), bad, pk, p)
    assert not any(res)


def test_verify_exhaustive_corruption_128f(eng, golden):
    """every single-byte corruption of a 128f signature fails."""
    p = derive("128f")
    sk = H(golden["sets"]["128f"]["keygen"]["sk"])
    pk = hs.PublicKey.from_bytes(sk[32:], p)
    sig = (GOLDEN_DIR / "sig_128f_zero.bin").read_bytes()
    bad = []
    for pos in range(len(sig)):
        b = bytearray(sig)
        b[pos] ^= 0xFF
        bad.append(bytes(b))
    res = hs.verify_batch([bytes(32)] * len(bad), bad, pk, p)
    assert not any(res)


@pytest.mark.parametrize("set_id", ("192f", "256f"))
def test_verify_every_byte_corrupted_batch(eng, oracle_mod, set_id):
    """Every byte position of a 192f / 256f signature corrupted once (one bit,
    a different bit per position), verified as one batch next to the intact
    signatures of a 64-message mixed batch: only the intact ones pass.
    Exercises every region's failure path (R, FORS leaves and auth, each
    layer's WOTS chains and auth) on the thread-local T_len verify kernel."""
    p = derive(set_id)
    rng = random.Random(606)
    sk = oracle_mod.keygen(set_id, rng.randbytes(3 * p.n))
    msgs = [rng.randbytes(rng.choice([0, 32, 100])) for _ in range(64)]
    eng.upload_keys(set_id, sk)
    sigs = eng.sign_batch(set_id, msgs)
    assert sigs[0] == oracle_mod.sign(set_id, sk, msgs[0])
    pk = sk[2 * p.n:]
    bad_msgs, bad_sigs = [], []
    for pos in range(p.sig_bytes):
        b = bytearray(sigs[pos % len(sigs)])
        b[pos] ^= 1 << (pos % 8)
        bad_msgs.append(msgs[pos % len(sigs)])
        bad_sigs.append(bytes(b))
    res = eng.verify_batch(set_id, pk, msgs + bad_msgs, sigs + bad_sigs)
    assert all(res[:len(msgs)])
    assert not any(res[len(msgs):]), [i for i, r in enumerate(res[len(msgs):]) if r][:10]


def test_errors(eng):
    p = derive("128f")
    with pytest.raises(hs.UsageError):
        hs.sign(b"x", hs.SecretKey.from_bytes(bytes(64), p), p, opt_rand=b"short")
    sk = hs.SecretKey.from_bytes(bytes(64), p)
    with pytest.raises(hs.UsageError):
        hs.sign_batch([b"a", b"b"], [sk], p, key_idx=[0, 3])
    with pytest.raises(hs.ConfigError):
        eng.set_config("128f", fors_trees_per_set=13, fors_sets_fused=1)  # 832 lanes > 768


@pytest.fixture(scope="module")
def config2(oracle_mod):
    p = derive("128f")
    rng = random.Random(2512_23969)
    sk = oracle_mod.keygen("128f", rng.randbytes(3 * p.n))
    msgs = [rng.randbytes(32) for _ in range(4096)]
    ref, _ = oracle_mod.sign_many("128f", sk, None, msgs)
    return sk, msgs, ref


@pytest.mark.parametrize("streams", [1, 3])
def test_config2_full_batch_128f(eng, config2, streams):
    """BASELINE config 2: 4096 messages, one key, every signature checked vs the
    CPU oracle; streams=3 splits the batch into uneven concurrent sub-graphs."""
    sk, msgs, ref = config2
    eng.upload_keys("128f", sk)
    base = eng.config("128f")
    try:
        eng.set_config("128f", streams=streams)
        sigs = eng.sign_batch("128f", msgs)
    finally:
        eng.set_config("128f", **base)
    assert sigs == ref
    assert all(eng.verify_batch("128f", sk[32:], msgs, sigs))


def test_graph_signer_stage_plugin(eng, oracle_mod):
    """The reference's stage-plugin protocol (batchgraph.py:93-131, 245-353) driven
    with random stage orders on 4 threads (tests/stage_driver.py; the reference's
    own scheduler runs the same plugin on CPU in test_tuner_config_graph.py): one
    GPU batch for all prepared messages, bytes == oracle, exact compression count."""
    from oracle_engine import oracle_wots_steps
    from stage_driver import drive, order_ok

    from paper_2512_23969_b200.batchgraph import GraphSigner

    p = derive("128f")
    rng = random.Random(11)
    sk_raw = oracle_mod.keygen("128f", rng.randbytes(48))
    sk = hs.SecretKey.from_bytes(sk_raw, p)
    msgs = [rng.randbytes(rng.choice([0, 32, 77])) for _ in range(24)]
    signer = GraphSigner(sk, p, engine=eng)
    sigs, log = drive(signer, msgs, workers=4, seed=3)
    assert order_ok(log, len(msgs))
    assert signer.launches == 1
    assert sigs == [oracle_mod.sign("128f", sk_raw, m) for m in msgs]
    assert signer.compressions == sum(hs.compressions_per_signature(
        p, len(m), digit_sum=oracle_wots_steps(oracle_mod, "128f", sk_raw, m))["total"] for m in msgs)


def test_config_apply_roundtrip(eng, tmp_path):
    from paper_2512_23969_b200.config import TuningConfig

    before = {s: eng.config(s) for s in SETS}
    cfg = TuningConfig.from_engine(eng)
    cfg.sets["192f"].b200.update(fors_trees_per_set=2, fors_sets_fused=4, fors_relax=True, streams=3)
    path = tmp_path / "t.json"
    cfg.save(path)
    try:
        TuningConfig.load(path).apply(eng)
        c = eng.config("192f")
        assert (c["fors_trees_per_set"], c["fors_sets_fused"], c["fors_relax"], c["streams"]) == (2, 4, True, 3)
    finally:
        for s, c in before.items():
            eng.set_config(s, **c)


@pytest.mark.parametrize("set_id", SETS)
def test_subtree_sharing(eng, oracle_mod, set_id):
    """Shared top-layer subtrees (0 .. max layers) with two keys in one batch: bytes == oracle."""
    p = derive(set_id)
    rng = random.Random(21 + p.n)
    sks = [oracle_mod.keygen(set_id, rng.randbytes(3 * p.n)) for _ in range(2)]
    count = 96
    msgs = [rng.randbytes(32) for _ in range(count)]
    kidx = [rng.randrange(2) for _ in range(count)]
    ref, _ = oracle_mod.sign_many(set_id, b"".join(sks), kidx, msgs)
    eng.upload_keys(set_id, sks)
    base = eng.config(set_id)
    top = 4 if set_id == "256f" else 6
    try:
        for L in range(top + 1):
            eng.set_config(set_id, shared_layers=L, shared_auto=False)
            assert eng.sign_batch(set_id, msgs, key_idx=kidx) == ref, L
            info = eng.batch_info(set_id)
            if info["shared_layers"]:
                # only the subtrees some message reads are built: <= one per (key, layer) per message
                assert 0 < info["shared_subtrees_built"] <= min(2 * hs.params.shared_units(p, info["shared_layers"]),
                                                                 count * info["shared_layers"])
        eng.set_config(set_id, shared_layers=top, shared_auto=True)
        assert eng.sign_batch(set_id, msgs, key_idx=kidx) == ref
        with pytest.raises(hs.ConfigError):
            eng.set_config(set_id, shared_layers=top + 1)
    finally:
        eng.set_config(set_id, **base)


def test_api_roundtrip_golden(eng, golden):
    """keygen -> sign -> verify through the public API on the reference's own
    192f vectors (sigcore.py:62-72, :139-178, :181-221)."""
    g = golden["sets"]["192f"]
    sk = hs.keygen("192f", bytes.fromhex(g["keygen"]["seed"]))
    assert sk.to_bytes().hex() == g["keygen"]["sk"]
    sig = hs.sign(bytes(32), sk, "192f")
    assert sig == (GOLDEN_DIR / "sig_192f_zero.bin").read_bytes()
    assert hs.verify(bytes(32), sig, sk.public(), "192f")
    assert not hs.verify(b"\x01" + bytes(31), sig, sk.public(), "192f")


@pytest.mark.parametrize("set_id", SETS)
def test_batch_size_rules(eng, oracle_mod, set_id):
    """The batch-size rules of the engine (batch_config): graphs of at most
    fors_small_batch messages run FORS_Sign with one tree per CTA, graphs of
    at most tree_small_batch messages reduce subtrees with warp shuffles
    (tree_split 1), graphs of at most `overlap` (>= 2) messages run the FORS /
    TREE / shared branches concurrently, larger ones in one stream order.  Counts on both sides of
    each threshold, with Relax on and off, sign the oracle's bytes."""
    p = derive(set_id)
    rng = random.Random(4242)
    sks = [oracle_mod.keygen(set_id, rng.randbytes(3 * p.n)) for _ in range(2)]
    msgs = [rng.randbytes(rng.choice([0, 32, 90])) for _ in range(21)]
    kidx = [rng.randrange(2) for _ in msgs]
    ref, _ = oracle_mod.sign_many(set_id, b"".join(sks), kidx, msgs)
    eng.upload_keys(set_id, sks)
    base = eng.config(set_id)
    try:
        for relax in (False, True):
            for small, tsmall, ov in ((20, 0, 0), (21, 21, 20), (0, 20, 21), (21, 64, 1), (64, 0, 0)):
                eng.set_config(set_id, fors_relax=relax, fors_small_batch=small, tree_small_batch=tsmall, overlap=ov,
                               streams=1, tree_split=2)
                for n in (1, 20, 21):
                    assert eng.sign_batch(set_id, msgs[:n], key_idx=kidx[:n]) == ref[:n], (relax, small, ov, n)
                    # the staged graph took the shape the rule gives for n messages
                    assert eng.batch_info(set_id)["tree_split"] == (1 if n <= tsmall else 2), (tsmall, n)
    finally:
        eng.set_config(set_id, **base)
