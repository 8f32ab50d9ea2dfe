"""CPU checks for the tuner (Algorithm 1), the config JSON and the task-graph scheduler.

Acceptance values from the reference SPEC.
"""

from __future__ import annotations

import json
from pathlib import Path
import random
import threading

import pytest

from conftest import SETS

from paper_2512_23969_b200.batchgraph import GraphSigner
from paper_2512_23969_b200.sigcore import SecretKey
from stage_driver import drive, order_ok
from paper_2512_23969_b200 import tuner
from paper_2512_23969_b200.config import TuningConfig
from paper_2512_23969_b200.errors import ConfigError, FormatError, TuningError, UsageError
from paper_2512_23969_b200.params import derive


def test_table3_reproduction():
    r128 = tuner.tree_tune(tuner.TuneInput(derive("128f"))).best
    assert (r128.lanes_per_set, r128.sets_fused, r128.lane_utilization, r128.scratch_utilization) == (704, 3, 0.6875,
                                                                                                     0.6875)
    r192 = tuner.tree_tune(tuner.TuneInput(derive("192f"))).best
    assert (r192.lanes_per_set, r192.sets_fused, r192.lane_utilization, r192.scratch_utilization) == (768, 2, 0.75, 0.75)


@pytest.mark.parametrize("set_id", SETS)
def test_candidates_feasible(set_id):
    inp = tuner.TuneInput(derive(set_id), seme_per_block=232448)
    res = tuner.tree_tune(inp)
    assert res.candidates and all(tuner.is_feasible(c, inp) for c in res.candidates)
    assert res.best == min(res.candidates, key=lambda c: c.sort_key(inp.params))


def test_tune_infeasible():
    with pytest.raises(TuningError):
        tuner.tree_tune(tuner.TuneInput(derive("256f"), seme_per_block=1024))


def test_padding_and_occupancy():
    assert [(s.banks_per_access, s.lane_interval, s.rows_per_region) for s in map(tuner.padding_solve, (16, 24, 32))] \
        == [(4, 8, 1), (6, 16, 3), (8, 4, 1)]
    assert abs(tuner.occupancy(65536, 64, 1024, 48) - 2 / 3) < 1e-9
    assert tuner.occupancy(65536, 128, 1024, 48) == 0
    with pytest.raises(UsageError):
        tuner.padding_solve(6)


def test_select_backends_tie_rule():
    runs = {}
    for k in tuner.KERNELS:
        for s in SETS:
            runs[(k, s)] = {"baseline": [1.0] * 10, "tuned": [0.99] * 10}
    runs[("TREE_Sign", "256f")]["tuned"] = [0.9] * 10
    sel = tuner.select_backends(runs)
    assert sel[("TREE_Sign", "256f")] == "tuned" and sel[("FORS_Sign", "128f")] == "baseline"
    del runs[("WOTS_Sign", "192f")]
    with pytest.raises(TuningError):
        tuner.select_backends(runs)


@pytest.mark.parametrize("set_id", SETS)
def test_device_candidates_respect_smem(set_id):
    from paper_2512_23969_b200 import _lib

    if not _lib.LIB_PATH.exists():
        _lib.build_native()
    cands = tuner.device_candidates(set_id, smem_optin=232448)
    assert cands
    p = derive(set_id)
    for c in cands:
        assert c.smem_bytes <= 232448 and c.lanes <= 768
        assert c.lanes == c.trees_per_set * (p.fors_t // 2 if c.relax else p.fors_t)
    assert cands == sorted(cands, key=tuner.DeviceCandidate.key)


def test_config_roundtrip(tmp_path):
    cfg = TuningConfig.default()
    cfg.validate()
    path = tmp_path / "cfg.json"
    cfg.save(path)
    back = TuningConfig.load(path)
    assert back.to_dict() == cfg.to_dict()
    # reference-format file (no "b200" block) loads too
    raw = json.loads(path.read_text())
    for row in raw["sets"].values():
        row.pop("b200")
    path.write_text(json.dumps(raw))
    ref = TuningConfig.load(path)
    assert ref.sets["128f"].fusion.lanes_per_set == 704 and not ref.sets["128f"].b200
    path.write_text("{")
    with pytest.raises(FormatError):
        TuningConfig.load(path)
    bad = cfg.to_dict()
    bad["sets"]["128f"]["b200"]["fors_trees_per_set"] = 40
    with pytest.raises(ConfigError):
        TuningConfig.from_dict(bad)


def test_pick_path_tie_rule():
    names = ("native", "fast", "mx248")
    assert tuner.pick_path({"native": 10.0, "fast": 9.0, "mx248": 8.0}, names) == 2
    assert tuner.pick_path({"native": 10.0, "fast": 9.9, "mx248": 9.85}, names) == 0  # within 2 %: keep native
    assert tuner.pick_path({"native": 10.0, "fast": 9.7, "mx248": 12.0}, names) == 1
    with pytest.raises(TuningError):
        tuner.pick_path({"native": 10.0}, names)


def test_shipped_tuned_config_is_loadable_and_in_range():
    """b200_tuned.json (the engine's default tuning) validates, and its SHA-path
    ids and FORS / TREE_Sign shape fields are legal for the built library."""
    from paper_2512_23969_b200 import _lib

    path = Path(__file__).resolve().parent.parent / "paper_2512_23969_b200" / "b200_tuned.json"
    cfg = TuningConfig.load(path)
    cfg.validate()
    n_paths = len(_lib.variant_names())
    for set_id, row in cfg.sets.items():
        b = row.b200
        assert all(0 <= v < n_paths for v in b["variant"].values()), (set_id, b["variant"])
        assert -1 <= b.get("fors_cta_levels", -1) <= derive(set_id).log_t
        assert b.get("tree_split", 1) in (0, 1, 2)
        assert int(b.get("overlap", 1)) >= 0 and int(b.get("fors_small_batch", 0)) >= 0
        assert int(b.get("tree_small_batch", 0)) >= 0


class _FakeSigner:
    """Stage bodies that record order; bytes depend only on the message."""

    sig_bytes = 8

    def __init__(self, fail_on=None):
        self.fail_on = fail_on
        self.order = []
        self.lock = threading.Lock()

    def prepare(self, msg, buffer):
        return type("Plan", (), {"msg": msg, "buffer": buffer, "f": False, "t": False})()

    def run_fors(self, plan):
        with self.lock:
            self.order.append(("F", plan.msg))
        plan.f = True

    def run_tree(self, plan):
        if self.fail_on is not None and plan.msg == self.fail_on:
            raise RuntimeError("boom")
        with self.lock:
            self.order.append(("T", plan.msg))
        plan.t = True

    def run_wots(self, plan):
        assert plan.f and plan.t
        plan.buffer[:] = (sum(plan.msg) & 0xFF).to_bytes(1, "big") * 8


def test_stage_driver_properties():
    """The test-side protocol driver (tests/stage_driver.py) honours the DAG and
    is deterministic in bytes across worker counts and random stage orders."""
    msgs = [bytes([i]) * 3 for i in range(12)]
    base, _ = drive(_FakeSigner(), msgs, workers=1)
    seen_orders = set()
    for trial in range(40):
        signer = _FakeSigner()
        sigs, log = drive(signer, msgs, workers=random.choice([2, 4, 8]), seed=trial)
        assert sigs == base and order_ok(log, len(msgs))
        first = {}
        for st, m in signer.order:
            first.setdefault(m, st)
        seen_orders |= set(first.values())
    assert seen_orders == {"F", "T"}
    with pytest.raises(RuntimeError):
        drive(_FakeSigner(fail_on=msgs[5]), msgs, workers=2)


REF_SRC = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not (REF_SRC / "herosign" / "batchgraph.py").exists(), reason="reference package absent")
def test_graph_signer_under_reference_scheduler(oracle_mod):
    """GraphSigner driven by the reference's OWN scheduler (build_graphs /
    execute_graphs / replay_check, batchgraph.py:110-242) through the stage
    plugin, with an oracle-backed engine stand-in (no GPU here): bytes equal the
    oracle, the reference's replay check holds, all buffers are allocated before
    launch, and the whole batch is one engine launch."""
    import sys

    sys.path.insert(0, str(REF_SRC))
    from herosign import batchgraph as ref_bg  # the reference itself, read-only

    from oracle_engine import OracleEngine

    p = derive("128f")
    rng = random.Random(11)
    sk_raw = oracle_mod.keygen("128f", rng.randbytes(48))
    msgs = [rng.randbytes(rng.choice([0, 32, 77])) for _ in range(12)]
    eng = OracleEngine(oracle_mod)
    signer = GraphSigner(SecretKey.from_bytes(sk_raw, p), p, engine=eng)
    graphs = ref_bg.build_graphs(msgs, 4, 3)
    pool = ref_bg.BufferPool()
    sigs, log = ref_bg.execute_graphs(graphs, 4, signer, pool=pool, rng=random.Random(3))
    assert ref_bg.replay_check(log, graphs)
    assert pool.allocations == len(msgs) and signer.launches == 1 and eng.sign_calls == 1
    assert sigs == [oracle_mod.sign("128f", sk_raw, m) for m in msgs]
    # the reference's own GraphSigner under the same scheduler: same bytes, and
    # its merged HashContext counter equals ours (batchgraph.py:279-285)
    from herosign import sigcore as ref_sigcore

    ref_signer = ref_bg.GraphSigner(ref_sigcore.SecretKey.from_bytes(sk_raw, ref_sigcore.derive("128f")), "128f")
    ref_sigs, _ = ref_bg.execute_graphs(ref_bg.build_graphs(msgs, 4, 3), 4, ref_signer)
    assert ref_sigs == sigs
    assert signer.compressions == ref_signer.compressions


def test_batch_size_rule_fields_validated(tmp_path):
    """The b200 row's batch-size thresholds (overlap, fors_small_batch,
    tree_small_batch) must be non-negative message counts."""
    path = Path(__file__).resolve().parent.parent / "paper_2512_23969_b200" / "b200_tuned.json"
    cfg = TuningConfig.load(path)
    assert cfg.sets["192f"].b200["overlap"] >= 2  # a threshold, not a flag
    for key, bad in (("overlap", -1), ("fors_small_batch", "64"), ("tree_small_batch", -16)):
        data = cfg.to_dict()
        data["sets"]["128f"]["b200"][key] = bad
        with pytest.raises(ConfigError):
            TuningConfig.from_dict(data)
