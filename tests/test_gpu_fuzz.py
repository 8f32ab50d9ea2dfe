"""Randomised configurations (a short, fixed-seed slice of tools/fuzz_gpu.py):
random set, batch size, message lengths, keys, opt_rand and engine shape per
iteration -- every signature must equal the oracle's and verify on the GPU."""

from __future__ import annotations

import importlib.util
import random
from pathlib import Path

import pytest

import paper_2512_23969_b200 as hs
from paper_2512_23969_b200.engine import variants
from paper_2512_23969_b200.tuner import device_candidates

pytestmark = pytest.mark.gpu

_spec = importlib.util.spec_from_file_location(
    "fuzz_gpu", Path(__file__).resolve().parent.parent / "tools" / "fuzz_gpu.py")
fuzz = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(fuzz)


@pytest.mark.parametrize("seed", range(48))
def test_random_configuration(oracle_mod, seed):
    eng = hs.get_engine()
    rng = random.Random(9_000_011 * (seed + 1))
    set_id = rng.choice(["128f", "192f", "256f"])
    p = hs.derive(set_id)
    cands = device_candidates(p, eng.device_info()["smem_optin"], alpha=0.0)
    cfg = fuzz.random_config(rng, p, cands, len(variants()))
    nkeys = rng.choice([1, 2])
    sks = [oracle_mod.keygen(set_id, rng.randbytes(3 * p.n)) for _ in range(nkeys)]
    count = rng.choice([1, 3, 17, 65, 130])
    msgs = [rng.randbytes(rng.choice([0, 32, 65, 200])) for _ in range(count)]
    kidx = [rng.randrange(nkeys) for _ in range(count)]
    opts = [rng.randbytes(p.n) if rng.random() < 0.3 else None for _ in range(count)]
    base = eng.config(set_id)
    try:
        eng.set_config(set_id, **cfg)
        eng.upload_keys(set_id, sks)
        got = eng.sign_batch(set_id, msgs, key_idx=kidx, opt_rand=opts)
        assert all(eng.verify_batch(set_id, [sk[2 * p.n:] for sk in sks], msgs, got, key_idx=kidx))
    finally:
        eng.set_config(set_id, **base)
    orand = b"".join(o if o is not None else sks[kidx[i]][2 * p.n:3 * p.n] for i, o in enumerate(opts))
    ref, _ = oracle_mod.sign_many(set_id, b"".join(sks), kidx, msgs, orand)
    bad = [i for i in range(count) if got[i] != ref[i]]
    assert not bad, (cfg, bad[:5])
