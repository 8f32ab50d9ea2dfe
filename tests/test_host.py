"""CPU-only checks: parameter tables, the C-ABI surface, error mapping, work-unit formula."""

from __future__ import annotations

import ctypes
import hashlib
import os
import re
from pathlib import Path

import pytest

from conftest import ROOT, SETS

import paper_2512_23969_b200 as hs
from paper_2512_23969_b200 import _lib
from paper_2512_23969_b200.params import compressions_per_signature, derive


@pytest.fixture(scope="module")
def L():
    if not _lib.LIB_PATH.exists():
        _lib.build_native()
    return _lib.lib()


def test_header_symbols_exported(L):
    header = (ROOT / "include" / "herosign_b200.h").read_text()
    declared = set(re.findall(r"HS_API\s+[\w\s\*]*?\b(hs_\w+)\s*\(", header))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name


@pytest.mark.parametrize("set_id", SETS)
def test_params_match_reference_and_device(L, golden, set_id):
    ref = golden["sets"][set_id]["params"]
    p = derive(set_id)
    for k, v in ref.items():
        assert getattr(p, k) == v, k
    arr = (ctypes.c_int32 * 32)()
    n = L.hs_params(p.index, arr, 32)
    fields = ("n h d log_t k w lg_w len1 len2 wots_len subtree_height subtree_leaves fors_t fors_msg_bytes "
              "tree_bits tree_bytes leaf_bits leaf_bytes digest_bytes wots_sig_bytes fors_sig_bytes "
              "ht_sig_bytes sig_bytes").split()
    assert n == len(fields)
    for f, v in zip(fields, arr[:n]):
        assert getattr(p, f) == v, f


def test_signature_sizes():
    # SPEC.md:599
    assert [derive(s).sig_bytes for s in SETS] == [17088, 35664, 49856]


@pytest.mark.parametrize("set_id", SETS)
def test_work_unit_formula(golden, set_id):
    """compressions_per_signature reproduces the reference's HashContext counter."""
    g = golden["sets"][set_id]
    p = derive(set_id)
    assert g["wots_gen_leaf"]["compressions"] == p.wots_len * (1 + (p.w - 1)) + (22 + p.wots_len * p.n + 72) // 64
    for case in g["sign"]:
        mlen = len(bytes.fromhex(case["msg"]))
        c = compressions_per_signature(p, mlen, digit_sum=0)
        digit_sum = case["compressions"] - c["total"]
        assert digit_sum == int(digit_sum) and 0 <= digit_sum <= p.d * p.wots_len * (p.w - 1)
        exact = compressions_per_signature(p, mlen, digit_sum=int(digit_sum))
        assert exact["total"] == case["compressions"]


def test_fors_smem_accounting(L):
    # ping-pong regions: 1.5 t nodes per tree (0.75 t with relax)
    # + 64 bytes of per-message PRF / F prefix states + 10 x 32 bytes of per-level H prefix states
    head = 64 + 10 * 32
    assert hs.Engine.fors_smem_bytes("128f", 11, 3, False) == 33 * 96 * 16 + head
    assert hs.Engine.fors_smem_bytes("256f", 2, 2, True) == 4 * 384 * 32 + head


def test_no_device_fails_loudly(L):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(hs.HeroSignError):
        hs.Engine(0)
    with pytest.raises(hs.HeroSignError):
        hs.keygen("128f", bytes(48))


def test_key_layout_and_regions():
    p = derive("192f")
    raw = bytes(range(4 * p.n))
    sk = hs.SecretKey.from_bytes(raw, p)
    assert sk.to_bytes() == raw and sk.public().to_bytes() == raw[2 * p.n:]
    with pytest.raises(hs.FormatError):
        hs.SecretKey.from_bytes(raw[:-1], p)
    with pytest.raises(hs.FormatError):
        hs.PublicKey.from_bytes(raw, p)
    r = hs.signature_regions(p)
    assert r["randomizer"] == (0, 24) and r["auth[21]"][1] == p.sig_bytes
    with pytest.raises(hs.ConfigError):
        derive("128s")


def test_message_to_indices_lsb_first(golden):
    for set_id in SETS:
        for v in golden["sets"][set_id]["h_msg"]:
            assert hs.message_to_indices(bytes.fromhex(v["mhash"]), set_id) == v["indices"]


@pytest.mark.parametrize("set_id", SETS)
def test_subtree_work_matches_reference_counter(golden, set_id):
    from paper_2512_23969_b200.params import shared_units, subtree_compressions

    assert subtree_compressions(set_id) == golden["sets"][set_id]["tree_layer"]["compressions"]
    p = derive(set_id)
    assert shared_units(set_id, 0) == 0 and shared_units(set_id, 1) == 1
    assert shared_units(set_id, 2) == 1 + p.subtree_leaves


def test_compiled_sha_paths(L):
    """hs_variants reports native, fast and the Mx<mask> paths listed in hs_variants.h."""
    names = _lib.variant_names()
    assert names[:2] == ("native", "fast")
    hdr = (ROOT / "paper_2512_23969_b200" / "csrc" / "hs_variants.h").read_text()
    default = re.search(r"#define HS_MX_MASKS ([\d, ]+)", hdr).group(1)
    masks = [int(x) for x in default.split(",")]
    if not os.environ.get("HERO_SIGN_LIB"):
        assert names[2:] == tuple(f"mx{m & 255}" + (f"p{m >> 8}" if m >> 8 else "") for m in masks)
    assert all(re.fullmatch(r"mx\d+(p\d+)?", n) for n in names[2:])


@pytest.mark.parametrize("set_id", SETS)
def test_oracle_wots_steps_pinned(golden, oracle_mod, set_id):
    """The oracle's compression counter minus its k re-derived FORS secrets is the
    reference's default-path count (hashes.py:117-159), for every golden sign
    case: this pins the per-message WOTS step counts the tests derive from it."""
    from oracle_engine import oracle_wots_steps

    p = derive(set_id)
    for case in golden["sets"][set_id]["sign"]:
        msg = bytes.fromhex(case["msg"])
        opt = bytes.fromhex(case["opt_rand"]) if case["opt_rand"] else None
        steps = oracle_wots_steps(oracle_mod, set_id, bytes.fromhex(case["sk"]), msg, opt)
        assert compressions_per_signature(p, len(msg), digit_sum=steps)["total"] == case["compressions"]


def test_ctx_out_exact_on_engine(golden, oracle_mod):
    """sigcore's ctx_out path (sign_on_engine) turns the engine's per-message WOTS
    step counts into SignContext.compressions equal to the reference's count."""
    from oracle_engine import OracleEngine

    from paper_2512_23969_b200.sigcore import SecretKey, sign_on_engine

    eng = OracleEngine(oracle_mod)
    for set_id in SETS:
        p = derive(set_id)
        for case in golden["sets"][set_id]["sign"]:
            ctx = []
            opt = [bytes.fromhex(case["opt_rand"])] if case["opt_rand"] else None
            sig = sign_on_engine(eng, [bytes.fromhex(case["msg"])], SecretKey.from_bytes(bytes.fromhex(case["sk"]), p),
                                 p, opt_rand=opt, ctx_out=ctx)[0]
            assert hashlib.sha256(sig).hexdigest() == case["sig_sha256"]
            assert ctx[0].compressions == case["compressions"], (set_id, case["tag"])
