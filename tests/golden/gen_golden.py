"""Generate golden fixtures by executing the reference package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/gen_golden.py

It imports the reference's pure-Python ``herosign`` package from
``/root/reference/pkg/src`` (stdlib only) and records inputs/outputs of every
function on the signing path into ``tests/golden/golden.json`` plus the full
deterministic signatures as ``sig_<set>_zero.bin``.  The GPU box has no
``/root/reference``; tests there read only these committed fixtures.
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
SEED = 2512_23969


def main() -> None:
    sys.path.insert(0, str(REF))
    from herosign import backends, hashes, params, sigcore, vexec, wots  # noqa: E402
    from herosign.address import ADDR_HASHTREE, Address  # noqa: E402
    from herosign.oracle import fors_sign  # noqa: E402

    rng = random.Random(SEED)
    golden: dict = {"source": "reference herosign (pkg/src/herosign), executed by gen_golden.py", "sets": {}}

    # -- SHA-256 (backends.py) -------------------------------------------
    sha = []
    for msg in (b"", b"abc", b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq", bytes(55), bytes(56),
                bytes(64), bytes(range(200))):
        sha.append({"msg": msg.hex(), "digest": backends.sha256_digest(msg).hex()})
    comp = []
    for _ in range(8):
        st = tuple(rng.getrandbits(32) for _ in range(8))
        blk = rng.randbytes(64)
        comp.append({"state": list(st), "block": blk.hex(), "out": list(backends.compress_baseline(st, blk))})
    golden["sha256"] = sha
    golden["compress"] = comp

    for set_id in ("128f", "192f", "256f"):
        p = params.derive(set_id)
        n = p.n
        g: dict = {"params": {k: getattr(p, k) for k in p.__dataclass_fields__ if k != "id"}}

        # thash / prf on assorted addresses and lengths (hashes.py:124-150)
        th, pr = [], []
        for mult in (1, 2, 3, p.wots_len, p.k):
            pk_seed = rng.randbytes(n)
            a = Address(bytearray(rng.randbytes(22)))
            msg = rng.randbytes(mult * n)
            ctx = hashes.HashContext(p, pk_seed)
            th.append({"pk_seed": pk_seed.hex(), "adrs": a.to_bytes().hex(), "msg": msg.hex(),
                       "out": ctx.thash(a, msg).hex()})
        for _ in range(4):
            sk_seed = rng.randbytes(n)
            a = Address(bytearray(rng.randbytes(22)))
            ctx = hashes.HashContext(p, rng.randbytes(n), sk_seed)
            pr.append({"sk_seed": sk_seed.hex(), "adrs": a.to_bytes().hex(), "out": ctx.prf(a).hex()})
        g["thash"], g["prf"] = th, pr

        # prf_msg / h_msg / indices (hashes.py:152-191, sigcore.py:75-90)
        pm, hm = [], []
        for mlen in (0, 1, 31, 32, 33, 55, 64, 100, 247):
            sk_prf, opt, msg = rng.randbytes(n), rng.randbytes(n), rng.randbytes(mlen)
            ctx = hashes.HashContext(p, rng.randbytes(n))
            pm.append({"sk_prf": sk_prf.hex(), "opt_rand": opt.hex(), "msg": msg.hex(),
                       "out": ctx.prf_msg(sk_prf, opt, msg).hex()})
            R, pk_seed, pk_root = rng.randbytes(n), rng.randbytes(n), rng.randbytes(n)
            mhash, tree, leaf = ctx.h_msg(R, pk_seed, pk_root, msg)
            hm.append({"R": R.hex(), "pk_seed": pk_seed.hex(), "pk_root": pk_root.hex(), "msg": msg.hex(),
                       "mhash": mhash.hex(), "tree": tree, "leaf": leaf,
                       "indices": sigcore.message_to_indices(mhash, p)})
        g["prf_msg"], g["h_msg"] = pm, hm

        # chain lengths (wots.py:33-39)
        cl = []
        for v in (bytes(n), b"\xff" * n, rng.randbytes(n), rng.randbytes(n)):
            cl.append({"msg_n": v.hex(), "lengths": wots.chain_lengths(v, p)})
        g["chain_lengths"] = cl

        # one WOTS leaf with its compression count (wots.py:119-143)
        pk_seed, sk_seed = rng.randbytes(n), rng.randbytes(n)
        ta = Address()
        ta.set_layer(3)
        ta.set_tree(0x1234567 & ((1 << p.tree_bits) - 1))
        ta.set_type(ADDR_HASHTREE)
        ctx = hashes.HashContext(p, pk_seed, sk_seed)
        leaf = wots.wots_gen_leaf(ctx, ta, 5, hashes.KERNEL_TREE)
        g["wots_gen_leaf"] = {"pk_seed": pk_seed.hex(), "sk_seed": sk_seed.hex(), "layer": 3,
                              "tree": 0x1234567 & ((1 << p.tree_bits) - 1), "leaf": 5, "out": leaf.hex(),
                              "compressions": ctx.compressions}

        # one hypertree layer (vexec.py:492-551)
        layer, tree, leaf_idx = 7, rng.getrandbits(p.tree_bits - p.subtree_height * 7), 3
        ctx = hashes.HashContext(p, pk_seed, sk_seed)
        res = vexec.run_tree_layer(ctx, layer, tree, leaf_idx)
        g["tree_layer"] = {"pk_seed": pk_seed.hex(), "sk_seed": sk_seed.hex(), "layer": layer, "tree": tree,
                           "leaf": leaf_idx, "root": res.root.hex(), "auth": res.auth_path.hex(),
                           "compressions": ctx.compressions}

        # FORS (oracle.py:113-146)
        tree = rng.getrandbits(p.tree_bits)
        leaf_idx = rng.randrange(p.subtree_leaves)
        indices = [rng.randrange(p.fors_t) for _ in range(p.k)]
        wa = Address()
        wa.set_tree(tree)
        wa.set_type(0)
        wa.set_keypair(leaf_idx)
        ctx = hashes.HashContext(p, pk_seed, sk_seed)
        fsig, fpk = fors_sign(ctx, b"", indices, wa)
        g["fors"] = {"pk_seed": pk_seed.hex(), "sk_seed": sk_seed.hex(), "tree": tree, "leaf": leaf_idx,
                     "indices": indices, "sig_sha256": hashlib.sha256(fsig).hexdigest(), "pk": fpk.hex()}

        # WOTS sign of a value at one address (wots.py:68-82)
        msg_n = rng.randbytes(n)
        wa2 = Address()
        wa2.set_layer(2)
        wa2.set_tree(tree >> p.subtree_height)
        wa2.set_type(0)
        wa2.set_keypair(leaf_idx)
        ctx = hashes.HashContext(p, pk_seed, sk_seed)
        wsig = wots.wots_sign(ctx, msg_n, wa2)
        g["wots_sign"] = {"pk_seed": pk_seed.hex(), "sk_seed": sk_seed.hex(), "layer": 2,
                          "tree": tree >> p.subtree_height, "keypair": leaf_idx, "msg_n": msg_n.hex(),
                          "sig": wsig.hex()}

        # keygen + full signatures (sigcore.py:62-178); the default (parallel) path
        seed0 = bytes(range(3 * n))
        sk0 = sigcore.keygen(p, seed0)
        signs = []
        cases = [(sk0, bytes(32), None, "zero"), (sk0, b"abc", b"\xa5" * n, "abc")]
        keys = [sigcore.keygen(p, rng.randbytes(3 * n)) for _ in range(2)]
        for i, mlen in enumerate((0, 1, 32, 77, 200)):
            cases.append((keys[i % 2], rng.randbytes(mlen), rng.randbytes(n) if i % 2 else None, f"rand{i}"))
        for sk, msg, opt, tag in cases:
            ctxs: list = []
            sig = sigcore.sign(msg, sk, p, opt_rand=opt, ctx_out=ctxs)
            assert sigcore.verify(msg, sig, sk.public(), p)
            signs.append({"tag": tag, "sk": sk.to_bytes().hex(), "msg": msg.hex(),
                          "opt_rand": opt.hex() if opt is not None else None,
                          "sig_sha256": hashlib.sha256(sig).hexdigest(), "compressions": ctxs[0].compressions})
            if tag == "zero":
                (OUT / f"sig_{set_id}_zero.bin").write_bytes(sig)
        g["keygen"] = {"seed": seed0.hex(), "sk": sk0.to_bytes().hex()}
        g["sign"] = signs

        # the bench recipe: first messages of the synthetic batch
        brng = random.Random(SEED)
        bsk = sigcore.keygen(p, brng.randbytes(3 * n))
        bmsgs = [brng.randbytes(32) for _ in range(3)]
        g["bench_recipe"] = {"sk": bsk.to_bytes().hex(),
                             "sig_sha256": [hashlib.sha256(sigcore.sign(m, bsk, p)).hexdigest() for m in bmsgs]}
        golden["sets"][set_id] = g
        print(set_id, "done", file=sys.stderr)

    (OUT / "golden.json").write_text(json.dumps(golden, indent=1) + "\n")


if __name__ == "__main__":
    main()
