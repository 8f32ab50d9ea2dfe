"""Pin the C oracle (oracle/hs_oracle.c) against the reference's own outputs.

Fixtures come from tests/golden/gen_golden.py, which executes the reference
package.  Both SHA-256 compressions of the oracle (scalar and SHA-NI) are
checked, mirroring the reference's two backends (backends.py:51-123).
"""

from __future__ import annotations

import hashlib

import pytest

from conftest import GOLDEN_DIR, SETS

H = bytes.fromhex


@pytest.fixture(params=["native", "scalar"])
def orc(request, oracle_mod):
    oracle_mod.force_scalar(request.param == "scalar")
    yield oracle_mod
    oracle_mod.force_scalar(False)


def test_sha256_vectors(orc, golden):
    for v in golden["sha256"]:
        assert orc.sha256(H(v["msg"])).hex() == v["digest"]
    for v in golden["compress"]:
        assert list(orc.compress(tuple(v["state"]), H(v["block"]))) == v["out"]


@pytest.mark.parametrize("set_id", SETS)
def test_params(oracle_mod, golden, set_id):
    ref = golden["sets"][set_id]["params"]
    mine = oracle_mod.params(set_id)
    for k, v in mine.items():
        alias = {"hp": "subtree_height", "leaves": "subtree_leaves", "t": "fors_t"}.get(k, k)
        assert ref[alias] == v, k


@pytest.mark.parametrize("set_id", SETS)
def test_primitives(orc, golden, set_id):
    g = golden["sets"][set_id]
    for v in g["thash"]:
        assert orc.thash(set_id, H(v["pk_seed"]), H(v["adrs"]), H(v["msg"])).hex() == v["out"]
    for v in g["prf"]:
        assert orc.prf(set_id, H(v["sk_seed"]), H(v["adrs"])).hex() == v["out"]
    for v in g["prf_msg"]:
        assert orc.prf_msg(set_id, H(v["sk_prf"]), H(v["opt_rand"]), H(v["msg"])).hex() == v["out"]
    for v in g["h_msg"]:
        mh, tree, leaf = orc.h_msg(set_id, H(v["R"]), H(v["pk_seed"]), H(v["pk_root"]), H(v["msg"]))
        assert (mh.hex(), tree, leaf) == (v["mhash"], v["tree"], v["leaf"])
        assert orc.message_to_indices(set_id, mh) == v["indices"]
    for v in g["chain_lengths"]:
        assert orc.chain_lengths(set_id, H(v["msg_n"])) == v["lengths"]


@pytest.mark.parametrize("set_id", SETS)
def test_components(orc, golden, set_id):
    g = golden["sets"][set_id]
    v = g["wots_gen_leaf"]
    leaf, comps = orc.wots_gen_leaf(set_id, H(v["pk_seed"]), H(v["sk_seed"]), v["layer"], v["tree"], v["leaf"])
    assert leaf.hex() == v["out"] and comps == v["compressions"]
    v = g["tree_layer"]
    root, auth = orc.tree_layer(set_id, H(v["pk_seed"]), H(v["sk_seed"]), v["layer"], v["tree"], v["leaf"])
    assert root.hex() == v["root"] and auth.hex() == v["auth"]
    v = g["fors"]
    sig, pk = orc.fors_sign(set_id, H(v["pk_seed"]), H(v["sk_seed"]), v["tree"], v["leaf"], v["indices"])
    assert hashlib.sha256(sig).hexdigest() == v["sig_sha256"] and pk.hex() == v["pk"]
    v = g["wots_sign"]
    sig = orc.wots_sign(set_id, H(v["pk_seed"]), H(v["sk_seed"]), v["layer"], v["tree"], v["keypair"], H(v["msg_n"]))
    assert sig.hex() == v["sig"]


@pytest.mark.parametrize("set_id", SETS)
def test_keygen_sign_verify(oracle_mod, golden, set_id):
    g = golden["sets"][set_id]
    assert oracle_mod.keygen(set_id, H(g["keygen"]["seed"])).hex() == g["keygen"]["sk"]
    n = oracle_mod.params(set_id)["n"]
    for v in g["sign"]:
        sk = H(v["sk"])
        opt = H(v["opt_rand"]) if v["opt_rand"] else None
        sig = oracle_mod.sign(set_id, sk, H(v["msg"]), opt)
        assert hashlib.sha256(sig).hexdigest() == v["sig_sha256"], v["tag"]
        assert oracle_mod.verify(set_id, sk[2 * n:], H(v["msg"]), sig)
        if v["tag"] == "zero":
            assert sig == (GOLDEN_DIR / f"sig_{set_id}_zero.bin").read_bytes()


def test_verify_rejects_corruption(oracle_mod):
    """SPEC.md:601 style: corrupt bytes across every region of a 128f signature."""
    sig = (GOLDEN_DIR / "sig_128f_zero.bin").read_bytes()
    import json
    g = json.loads((GOLDEN_DIR / "golden.json").read_text())["sets"]["128f"]
    pk = H(g["keygen"]["sk"])[32:]
    assert oracle_mod.verify("128f", pk, bytes(32), sig)
    for pos in range(0, len(sig), 97):
        bad = bytearray(sig)
        bad[pos] ^= 0x01
        assert not oracle_mod.verify("128f", pk, bytes(32), bytes(bad)), pos
    assert not oracle_mod.verify("128f", pk, bytes(32), sig[:-1])


def test_sign_many_matches_single(oracle_mod, golden):
    g = golden["sets"]["128f"]
    sk = H(g["keygen"]["sk"])
    msgs = [bytes(32), b"abc", b""]
    sigs, comps = oracle_mod.sign_many("128f", sk, None, msgs, threads=3)
    for m, s in zip(msgs, sigs):
        assert s == oracle_mod.sign("128f", sk, m)
    assert comps > 3 * 113000
