"""ncu target: sign `count` messages, then one GPU verification of them (128f by default)."""
from __future__ import annotations

import argparse
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2512_23969_b200 as hs  # noqa: E402
from paper_2512_23969_b200.engine import PinnedBuffer, pack_messages  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--set", dest="set_id", default="128f")
ap.add_argument("--count", type=int, default=65536)
a = ap.parse_args()
eng = hs.get_engine(0)
p = hs.derive(a.set_id)
rng = random.Random(5)
sk = eng.keygen_batch(a.set_id, [rng.randbytes(3 * p.n)])[0]
eng.upload_keys(a.set_id, sk)
blob, offs = pack_messages([rng.randbytes(32) for _ in range(a.count)])
out = PinnedBuffer(a.count * p.sig_bytes)
eng.sign_into(a.set_id, blob, offs, a.count, out.ptr)
ok = eng.verify_into(a.set_id, sk[2 * p.n:], blob, offs, a.count, out.ptr)
print("verified", int(ok.sum()), "of", a.count)
out.free()
