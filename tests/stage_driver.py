"""Test-side driver of the reference's stage-plugin protocol.

The reference drives a duck-typed signer (``sig_bytes``,
``prepare(msg, buffer) -> plan``, ``run_fors / run_tree / run_wots(plan)``)
from its task-graph scheduler (reference batchgraph.py:93-131, 124-226): every
output buffer is allocated and every message prepared before the first stage
runs, FORS and TREE of a message run in either order on any worker, and WOTS
runs after both.  On the GPU box the reference package is absent, so the GPU
tests drive ``GraphSigner`` with this small independent driver of the same
protocol; on the CPU box ``test_tuner_config_graph.py`` runs the reference's
own ``execute_graphs`` as well.  Test infrastructure only.
"""

from __future__ import annotations

import random
import threading


def drive(signer, msgs, workers: int = 4, seed: int = 0):
    """Run the protocol over ``msgs`` with ``workers`` threads picking ready
    stages at random.  Returns (signatures in message order, stage log as
    (message index, stage) in completion order)."""
    rng = random.Random(seed)
    plans = [signer.prepare(m, bytearray(signer.sig_bytes)) for m in msgs]  # all buffers before launch
    ready = [(i, s) for i in range(len(msgs)) for s in ("FORS", "TREE")]
    done_parts = [set() for _ in msgs]
    log, errors = [], []
    left = 3 * len(msgs)
    cv = threading.Condition()

    def worker():
        nonlocal left
        while True:
            with cv:
                while not ready and left > 0 and not errors:
                    cv.wait()
                if left <= 0 or errors:
                    cv.notify_all()
                    return
                i, stage = ready.pop(rng.randrange(len(ready)))
            try:
                getattr(signer, f"run_{stage.lower()}")(plans[i])
            except Exception as exc:  # surfaced after join
                with cv:
                    errors.append(exc)
                    cv.notify_all()
                return
            with cv:
                log.append((i, stage))
                left -= 1
                done_parts[i].add(stage)
                if stage != "WOTS" and done_parts[i] >= {"FORS", "TREE"}:
                    ready.append((i, "WOTS"))
                cv.notify_all()

    threads = [threading.Thread(target=worker) for _ in range(max(1, workers))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return [bytes(p.buffer) for p in plans], log


def order_ok(log, n: int) -> bool:
    """Each message ran FORS, TREE and WOTS once, WOTS last."""
    pos = {}
    for k, (i, s) in enumerate(log):
        if (i, s) in pos:
            return False
        pos[(i, s)] = k
    for i in range(n):
        if any((i, s) not in pos for s in ("FORS", "TREE", "WOTS")):
            return False
        if pos[(i, "WOTS")] < max(pos[(i, "FORS")], pos[(i, "TREE")]):
            return False
    return True
