"""Tree Tuning (Algorithm 1), padding solver, backend selection -- and the
on-device search that picks the FORS fusion layout and SHA-256 paths on the
B200 itself.

The pure functions restate the reference's tuner.py so its acceptance values
hold: ``tree_tune`` reproduces Table 3 at the
48 KB budget, ``padding_solve`` gives (4,8,1)/(6,16,3)/(8,4,1),
``occupancy`` the Eq. 1 estimate.  ``device_candidates`` re-runs the same
search against the B200 kernel's real shared-memory footprint
(``hs_fors_smem_bytes``) and the device's opt-in limit (227 KB), with and
without Relax, and ``tune_on_device`` times the best candidates and both
SHA-256 paths with CUDA events and keeps the fastest (the paper's
"near-optimal candidates ... selected based on empirical profiling",
PAPER.md:286).
"""

from __future__ import annotations

import math
import random
import statistics
from dataclasses import dataclass, field
from fractions import Fraction
from math import ceil, gcd

from .errors import TuningError, UsageError
from .params import PARAMETER_SETS, DerivedParams, derive

DEFAULT_SEME = 49152
DEFAULT_T_MAX = 1024
B200_FORS_MAX_LANES = 768  # csrc kForsMaxLanes: keeps 85 registers per lane
DEFAULT_ALPHA = 0.5
BANKS = 32
BANK_WIDTH = 4
TRANSACTION_BYTES = 128
KERNELS = ("FORS_Sign", "TREE_Sign", "WOTS_Sign")


@dataclass(frozen=True)
class TuneInput:
    params: DerivedParams
    seme_per_block: int = DEFAULT_SEME
    t_max: int = DEFAULT_T_MAX
    alpha: float = DEFAULT_ALPHA


@dataclass(frozen=True)
class FusionCandidate:
    """One feasible fusion shape (tuner.py:44-56)."""

    lanes_per_set: int
    sets_fused: int
    trees_per_set: int
    lane_utilization: float
    scratch_utilization: float
    sync_score: float

    def sort_key(self, p: DerivedParams):
        sync = Fraction(p.log_t * ceil(Fraction(p.k, self.trees_per_set)), self.sets_fused)
        return (sync, -self.lane_utilization, -self.scratch_utilization, self.lanes_per_set, self.sets_fused)


@dataclass(frozen=True)
class TuneResult:
    best: FusionCandidate
    candidates: list = field(default_factory=list)


def is_feasible(c: FusionCandidate, inp: TuneInput) -> bool:
    """Independent re-check of every predicate (tuner.py:65-88)."""
    p = inp.params
    t = p.fors_t
    if c.lanes_per_set % t or c.lanes_per_set > inp.t_max:
        return False
    if c.trees_per_set != c.lanes_per_set // t:
        return False
    s_used = c.sets_fused * c.trees_per_set * t * p.n
    if c.sets_fused < 1 or s_used >= inp.seme_per_block:
        return False
    if c.sets_fused > p.k // c.trees_per_set:
        return False
    u_t = c.lanes_per_set / inp.t_max
    u_s = s_used / inp.seme_per_block
    if u_t < inp.alpha or (u_t == 1.0 and u_s == 1.0):
        return False
    return (c.lane_utilization == u_t and c.scratch_utilization == u_s
            and c.sync_score == p.log_t * ceil(p.k / c.trees_per_set) / c.sets_fused)


def tree_tune(inp: TuneInput) -> TuneResult:
    """Algorithm 1 (tuner.py:91-143): arg-min (sync, -U_T, -U_S)."""
    p = inp.params
    t = p.fors_t
    s_tree = t * p.n
    if inp.seme_per_block < s_tree:
        raise TuningError(f"no tree fits: one {p.id} FORS tree needs {s_tree} scratch bytes, "
                          f"budget is {inp.seme_per_block}")
    cands, pruned = [], {"alpha": 0, "saturated": 0, "exact_fit": 0}
    for lanes in range(t, inp.t_max + 1, t):
        n_tree = lanes // t
        s_set = n_tree * s_tree
        if s_set > inp.seme_per_block:
            continue
        for f in range(1, min(inp.seme_per_block // s_set, p.k // n_tree) + 1):
            s_used = f * s_set
            u_t, u_s = lanes / inp.t_max, s_used / inp.seme_per_block
            if u_t == 1.0 and u_s == 1.0:
                pruned["saturated"] += 1
                continue
            if u_s == 1.0:
                pruned["exact_fit"] += 1
                continue
            if u_t < inp.alpha:
                pruned["alpha"] += 1
                continue
            cands.append(FusionCandidate(lanes, f, n_tree, u_t, u_s, p.log_t * ceil(p.k / n_tree) / f))
    if not cands:
        raise TuningError(f"no feasible fusion shape for {p.id} (budget {inp.seme_per_block}, t_max {inp.t_max}, "
                          f"alpha {inp.alpha}); pruned: {pruned}")
    return TuneResult(best=min(cands, key=lambda c: c.sort_key(p)), candidates=cands)


def occupancy(r_total: int, r_thread: int, t_block: int, w_max: int) -> float:
    """Eq. 1 register-limited occupancy (tuner.py:146-154)."""
    if min(r_total, r_thread, t_block, w_max) <= 0:
        raise UsageError("occupancy inputs must all be positive")
    return (r_total // (r_thread * t_block)) * (t_block / 32) / w_max


@dataclass(frozen=True)
class PaddingScheme:
    access_bytes: int
    banks_per_access: int
    lane_interval: float
    rows_per_region: int


def padding_solve(access_bytes: int) -> PaddingScheme:
    """Minimal solution of 128 R = B_n * 4 * T_h (Eq. 2/3; tuner.py:157-171)."""
    if access_bytes <= 0 or access_bytes % BANK_WIDTH:
        raise UsageError(f"access width must be a positive multiple of 4, got {access_bytes}")
    b_n = access_bytes // BANK_WIDTH
    r = b_n // gcd(TRANSACTION_BYTES // BANK_WIDTH, b_n)
    t_h = TRANSACTION_BYTES * r // (b_n * BANK_WIDTH)
    return PaddingScheme(access_bytes, b_n, t_h, r)


def _trimmed_mean(xs):
    if len(xs) < 3:
        return statistics.fmean(xs)
    s = sorted(xs)
    return statistics.fmean(s[1:-1])


def select_backends(profile_runs: dict, reps: int = 10, tie_tolerance: float = 0.02) -> dict:
    """Per (kernel, set) pick 'tuned' only if its trimmed mean beats 'baseline' by
    more than tie_tolerance (tuner.py:184-219).  Returns {(kernel, set): name}."""
    missing = []
    for kernel in KERNELS:
        for set_id in PARAMETER_SETS:
            cell = profile_runs.get((kernel, set_id))
            if cell is None or any(len(cell.get(b, ())) < reps for b in ("baseline", "tuned")):
                missing.append((kernel, set_id))
    if missing:
        raise TuningError(f"profile incomplete; uncovered cells: {sorted(set(missing))}")
    out = {}
    for kernel in KERNELS:
        for set_id in PARAMETER_SETS:
            cell = profile_runs[(kernel, set_id)]
            base, tuned = _trimmed_mean(cell["baseline"]), _trimmed_mean(cell["tuned"])
            out[(kernel, set_id)] = "tuned" if tuned < base * (1.0 - tie_tolerance) else "baseline"
    return out


def pick_path(cell_ms: dict, names, tie_tolerance: float = 0.02) -> int:
    """Variant id for one (kernel, set) cell of timings {path name: ms}: the
    fastest compiled SHA-256 path, but a non-native path replaces native only
    when it is faster by more than tie_tolerance (the reference's rule,
    tuner.py:206-218, generalised from two backends to the compiled list)."""
    names = list(names)
    missing = [n for n in names if n not in cell_ms]
    if missing:
        raise TuningError(f"no timing for SHA-256 paths {missing}")
    best = min(range(len(names)), key=lambda v: cell_ms[names[v]])
    return best if cell_ms[names[best]] < cell_ms["native"] * (1.0 - tie_tolerance) else 0


# ---------------------------------------------------------------------------
# B200: the same search over the real kernel footprint, then device timing
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class DeviceCandidate:
    trees_per_set: int
    sets_fused: int
    relax: bool
    lanes: int
    smem_bytes: int
    passes: int
    sync_score: float
    lane_utilization: float
    smem_utilization: float

    def key(self):
        return (self.sync_score, -self.lane_utilization, -self.smem_utilization, self.lanes, self.sets_fused)


def device_candidates(params, smem_optin: int, t_max: int = B200_FORS_MAX_LANES, alpha: float = DEFAULT_ALPHA,
                      smem_of=None) -> list[DeviceCandidate]:
    """Algorithm 1 over (N_tree, F, Relax) with the B200 kernel's smem formula.

    smem_of(set_id, n_tree, f, relax) -> bytes; defaults to the library's
    hs_fors_smem_bytes (ping-pong levels: 1.5 t nodes per tree, 0.75 t with
    Relax).  Barrier count per pass is log_t (log_t - 1 with Relax).
    """
    p = derive(params)
    if smem_of is None:
        from .engine import Engine

        smem_of = Engine.fors_smem_bytes
    out = []
    for relax in (False, True):
        lanes_per_tree = p.fors_t // 2 if relax else p.fors_t
        for n_tree in range(1, t_max // lanes_per_tree + 1):
            lanes = n_tree * lanes_per_tree
            sets_total = ceil(p.k / n_tree)
            for f in range(1, max(1, p.k // n_tree) + 1):
                smem = smem_of(p.id, n_tree, f, relax)
                if smem > smem_optin:
                    break
                u_t = lanes / t_max
                if u_t < alpha and not (n_tree * f >= p.k):
                    continue
                passes = ceil(sets_total / f)
                syncs = (p.log_t - (1 if relax else 0)) * passes
                out.append(DeviceCandidate(n_tree, f, relax, lanes, int(smem), passes, syncs / 1.0, u_t,
                                           smem / smem_optin))
    if not out:
        raise TuningError(f"no feasible B200 FORS layout for {p.id} under {smem_optin} bytes")
    return sorted(out, key=DeviceCandidate.key)


def _synthetic(engine, set_id: str, count: int):
    from .engine import pack_messages

    p = derive(set_id)
    rng = random.Random(2512_23969)
    seed = rng.randbytes(3 * p.n)
    sk = engine.keygen_batch(set_id, [seed])[0]
    engine.upload_keys(set_id, sk)
    msgs = [rng.randbytes(32) for _ in range(count)]
    blob, offs = pack_messages(msgs)
    engine.stage(set_id, blob, offs, count)


def _kernel_ms(engine, set_id: str, count: int, kernel: str, reps: int) -> list[float]:
    out = []
    for _ in range(reps):
        engine.bench_run(set_id, count, 1, 1, 0)
        out.append(engine.timings()[kernel])
    return out


def tune_on_device(engine, set_id: str, count: int = 2048, top: int = 12, reps: int = 5,
                   tie_tolerance: float = 0.02, tune_variants: bool = True) -> dict:
    """Search the FORS layout and per-kernel SHA-256 path on this device.

    1. ``device_candidates`` enumerates every layout Algorithm 1 admits at
       S_max = opt-in smem (both Relax modes); each is timed (FORS_Sign kernel,
       CUDA events, serial mode), the ``top`` fastest are re-timed and the best
       trimmed mean wins; then every split between in-CTA levels and the
       batch-wide level grids (``fors_cta_levels``) is timed for it.
    2. For each kernel every compiled SHA-256 path (engine.variants()) is timed;
       the fastest replaces 'native' only if it is faster by more than
       ``tie_tolerance`` (the reference's rule, tuner.py:206-218).
    3. Sub-batches per graph (T) and stream overlap (FORS_Sign || TREE_Sign and
       concurrent sub-batches, or one stream order) are timed end to end from
       pinned host buffers at ``count`` messages.
    4. The batch-size rules: the overlap threshold below ``count`` (when one
       stream order won), the largest graph that runs FORS_Sign with one tree
       per CTA (``fors_small_batch``) and the largest that reduces subtrees
       with warp shuffles (``tree_small_batch``), from graph device times.
    Returns the chosen config plus the timing table; the engine is left
    configured with it.
    """
    p = derive(set_id)
    info = engine.device_info()
    # Every feasible layout (no alpha pruning: small CTAs that share an SM hide
    # each other's sparse upper levels) is timed once; the `top` fastest are
    # re-timed with `reps` runs and the best trimmed mean wins.
    cands = device_candidates(p, info["smem_optin"], alpha=0.0)
    _synthetic(engine, set_id, count)
    base = engine.config(set_id)
    first = []
    for c in cands:
        engine.set_config(set_id, fors_trees_per_set=c.trees_per_set, fors_sets_fused=c.sets_fused,
                          fors_relax=c.relax)
        first.append((min(_kernel_ms(engine, set_id, count, "FORS_Sign", 2)), c))
    first.sort(key=lambda x: x[0])
    table = []
    for _, c in first[:top]:
        engine.set_config(set_id, fors_trees_per_set=c.trees_per_set, fors_sets_fused=c.sets_fused,
                          fors_relax=c.relax)
        ms = _trimmed_mean(_kernel_ms(engine, set_id, count, "FORS_Sign", reps))
        table.append({"trees_per_set": c.trees_per_set, "sets_fused": c.sets_fused, "relax": c.relax,
                      "lanes": c.lanes, "smem_bytes": c.smem_bytes, "passes": c.passes, "fors_ms": ms})
    best = min(table, key=lambda r: r["fors_ms"])
    engine.set_config(set_id, fors_trees_per_set=best["trees_per_set"], fors_sets_fused=best["sets_fused"],
                      fors_relax=best["relax"])
    # 1b. split between the CTA's in-shared-memory levels and the batch-wide
    #     level grids for the chosen layout (fors_cta_levels; -1 = auto)
    ltable = {}
    for lc in [-1] + list(range(1 if best["relax"] else 0, p.log_t + 1)):
        engine.set_config(set_id, fors_cta_levels=lc)
        ltable[lc] = _trimmed_mean(_kernel_ms(engine, set_id, count, "FORS_Sign", reps))
    best_lc = min(ltable, key=ltable.get)
    engine.set_config(set_id, fors_cta_levels=best_lc)
    best = dict(best, fors_cta_levels=best_lc, fors_ms=ltable[best_lc])
    variants = dict(base["variant"])
    vtable = {}
    if tune_variants:
        from .engine import variants as compiled_paths

        names = compiled_paths()
        for kernel in ("FORS_Sign", "TREE_Sign", "WOTS_Sign"):
            cell = {}
            for v, name in enumerate(names):
                var = dict(variants)
                var[kernel] = v
                engine.set_config(set_id, variant=var)
                cell[name] = _trimmed_mean(_kernel_ms(engine, set_id, count, kernel, reps))
            variants[kernel] = pick_path(cell, names, tie_tolerance)
            vtable[kernel] = cell
        engine.set_config(set_id, variant=variants)
    # 3. multi-stream batching: T prioritised sub-batches per graph, timed end to
    #    end (pinned host I/O: each sub-batch's D2H overlaps the others' compute)
    import time

    from .engine import PinnedBuffer, pack_messages

    rng = random.Random(7)
    msgs = [rng.randbytes(32) for _ in range(count)]
    blob, offs = pack_messages(msgs)
    out = PinnedBuffer(count * p.sig_bytes)
    stable = {}
    try:
        for T, ov in [(T, ov) for ov in (True, False) for T in (1, 2, 3, 4, 6, 8)]:
            engine.set_config(set_id, streams=T, overlap=ov)
            engine.sign_into(set_id, blob, offs, count, out.ptr)
            runs = []
            for _ in range(reps):
                t0 = time.perf_counter()
                engine.sign_into(set_id, blob, offs, count, out.ptr)
                runs.append(1e3 * (time.perf_counter() - t0))
            stable[T if ov else f"{T}/serial"] = _trimmed_mean(runs)
    finally:
        out.free()
    best_key = min(stable, key=stable.get)
    best_T = int(str(best_key).split("/")[0])
    best_ov = not str(best_key).endswith("/serial")
    engine.set_config(set_id, streams=best_T, overlap=best_ov, fors_small_batch=0, tree_small_batch=0)
    # 4. batch-size rules (the engine's batch_config), graph device time on
    #    smaller batches: (a) when one stream order won at `count`, the largest
    #    of count/2, count/4, ... (>= 16) at which the concurrent branches are
    #    faster becomes the overlap threshold; (b) one FORS tree per CTA and
    #    (c) the warp-shuffle Merkle reduction (tree_split 1 for a tree_split 2
    #    config) are each kept for graphs up to the largest of 16, 64, 256
    #    messages at which they win by more than tie_tolerance.
    def graph_ms(n: int, **kw) -> float:
        engine.set_config(set_id, **kw)
        _synthetic(engine, set_id, n)
        engine.bench_run(set_id, n, 2, 0)
        return _trimmed_mean(engine.bench_run(set_id, n, reps, 0))

    otable, small_table = {}, {}
    if not best_ov:
        n = count // 2
        while n >= 16:
            otable[n] = (graph_ms(n, overlap=1), graph_ms(n, overlap=0))
            if otable[n][0] < otable[n][1]:
                engine.set_config(set_id, overlap=n)
                break
            engine.set_config(set_id, overlap=0)
            n //= 2
    small = 0
    for n in (16, 64, 256):
        if n > count:
            break
        small_table[n] = (graph_ms(n, fors_small_batch=0), graph_ms(n, fors_small_batch=n))
        if not small_table[n][1] < small_table[n][0] * (1 - tie_tolerance):
            break
        small = n
    engine.set_config(set_id, fors_small_batch=small)
    tree_table, tsmall = {}, 0
    for n in (16, 64, 256):
        if n > count or engine.config(set_id)["tree_split"] != 2:
            break
        tree_table[n] = (graph_ms(n, tree_small_batch=0), graph_ms(n, tree_small_batch=n))
        if not tree_table[n][1] < tree_table[n][0] * (1 - tie_tolerance):
            break
        tsmall = n
    engine.set_config(set_id, tree_small_batch=tsmall)
    _synthetic(engine, set_id, count)
    return {"set": set_id, "count": count, "smem_optin": info["smem_optin"], "layouts": table,
            "best_layout": best, "cta_levels_ms": ltable, "variants": variants, "variant_ms": vtable,
            "streams_ms": stable, "overlap_ms": otable, "small_batch_ms": small_table,
            "tree_small_batch_ms": tree_table,
            "config": engine.config(set_id)}
