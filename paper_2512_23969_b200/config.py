"""Tuning configuration JSON (reference config.py:41-170), extended for B200.

The file keeps the reference's schema -- per set {fusion, padding, backends,
relax} plus seme_per_block / worker_width -- so a reference config loads
unchanged (its fusion / relax row then sets the FORS layout), and adds an
optional "b200" block per set carrying what the on-device tuner measured:
the kernel layout actually used (trees per set, fused sets, relax), the
SHA-256 path per kernel, WOTS-from-TREE and the batch chunk.  ``HERO_SIGN_CONFIG`` overrides the path as in the reference.
"""

from __future__ import annotations

import json
import os
import warnings
from dataclasses import dataclass, field
from pathlib import Path

from .errors import ConfigError, FormatError
from .params import PARAMETER_SETS, derive
from .tuner import (B200_FORS_MAX_LANES, DEFAULT_SEME, FusionCandidate, PaddingScheme, TuneInput, padding_solve,
                    tree_tune)

ENV_CONFIG_PATH = "HERO_SIGN_CONFIG"
DEFAULT_WORKERS = 4
KERNELS = ("FORS_Sign", "TREE_Sign", "WOTS_Sign")
MAX_VARIANTS = 64  # variant ids are checked against the built library by hs_config_set
MAX_LANES = 1024

# Engine defaults (csrc/hs_api.cu default_config); tune_on_device refines them.
B200_DEFAULTS = {
    "128f": {"fors_trees_per_set": 11, "fors_sets_fused": 3, "fors_relax": False},
    "192f": {"fors_trees_per_set": 3, "fors_sets_fused": 8, "fors_relax": False},
    "256f": {"fors_trees_per_set": 3, "fors_sets_fused": 6, "fors_relax": True},
}


@dataclass
class SetConfig:
    fusion: FusionCandidate
    padding: PaddingScheme
    backends: dict
    relax: bool
    b200: dict = field(default_factory=dict)


@dataclass
class TuningConfig:
    seme_per_block: int = DEFAULT_SEME
    worker_width: int = DEFAULT_WORKERS
    sets: dict = field(default_factory=dict)

    @classmethod
    def default(cls, seme: int = DEFAULT_SEME, alpha: float = 0.5) -> "TuningConfig":
        sets = {}
        for set_id in PARAMETER_SETS:
            p = derive(set_id)
            best = tree_tune(TuneInput(p, seme_per_block=seme, alpha=alpha)).best
            tuned_all = set_id == "256f"  # reference BackendSelection.default (backends.py:230-238)
            backends = {"FORS_Sign": "tuned", "TREE_Sign": "tuned" if tuned_all else "baseline",
                        "WOTS_Sign": "tuned" if tuned_all else "baseline"}
            b200 = dict(B200_DEFAULTS[set_id])
            b200.update({"variant": {k: 0 for k in KERNELS}, "wots_from_tree": True, "chunk": 16384, "streams": 1,
                         "shared_layers": 4 if set_id == "256f" else 6, "shared_auto": True})
            sets[set_id] = SetConfig(best, padding_solve(p.n), backends, set_id == "256f", b200)
        return cls(seme_per_block=seme, sets=sets)

    def validate(self) -> None:
        if self.worker_width < 1:
            raise ConfigError(f"worker width must be >= 1, got {self.worker_width}")
        if set(self.sets) != set(PARAMETER_SETS):
            raise ConfigError(f"config must cover exactly {sorted(PARAMETER_SETS)}, got {sorted(self.sets)}")
        for set_id, cfg in self.sets.items():
            p = derive(set_id)
            c = cfg.fusion
            if c.lanes_per_set != c.trees_per_set * p.fors_t or c.lanes_per_set > MAX_LANES:
                raise ConfigError(f"{set_id}: lanes_per_set {c.lanes_per_set} inconsistent")
            if cfg.padding.access_bytes != p.n:
                raise ConfigError(f"{set_id}: padding solved for {cfg.padding.access_bytes}-byte accesses")
            unknown = set(cfg.backends) - set(KERNELS)
            if unknown:
                raise ConfigError(f"{set_id}: unknown kernels {sorted(unknown)}")
            for k, v in cfg.backends.items():
                if v not in ("baseline", "tuned"):
                    raise ConfigError(f"{set_id}: backend {v!r} for {k}")
            b = cfg.b200
            if b:
                lanes = b.get("fors_trees_per_set", 1) * (p.fors_t // 2 if b.get("fors_relax") else p.fors_t)
                if lanes > MAX_LANES:
                    raise ConfigError(f"{set_id}: B200 layout needs {lanes} lanes")
                for k, v in b.get("variant", {}).items():
                    if k not in KERNELS + ("host",) or not (isinstance(v, int) and 0 <= v < MAX_VARIANTS):
                        raise ConfigError(f"{set_id}: bad variant {k}={v}")
                # batch-size rules: message-count thresholds (overlap also 0 / 1 / true / false)
                for k in ("overlap", "fors_small_batch", "tree_small_batch"):
                    if k in b and not (isinstance(b[k], int) and int(b[k]) >= 0):
                        raise ConfigError(f"{set_id}: {k} must be a message count >= 0, got {b[k]!r}")

    # -- engine binding --------------------------------------------------
    def apply(self, engine) -> None:
        """Push every set's B200 row into an Engine (hs_config_set)."""
        for set_id, cfg in self.sets.items():
            b = dict(cfg.b200) if cfg.b200 else {}
            if not b:
                # a reference config (no b200 block): its layout row drives the
                # FORS kernel -- N_tree and F from `fusion`, Relax from `relax`
                # (config.py:33-38) -- when the B200 kernel can run it (lanes
                # within its 768-lane CTA), else the engine keeps its layout
                p = derive(set_id)
                lanes = cfg.fusion.trees_per_set * (p.fors_t // 2 if cfg.relax else p.fors_t)
                if lanes <= B200_FORS_MAX_LANES:
                    b = {"fors_trees_per_set": cfg.fusion.trees_per_set, "fors_sets_fused": cfg.fusion.sets_fused,
                         "fors_relax": bool(cfg.relax)}
                else:
                    warnings.warn(f"{set_id}: reference layout {cfg.fusion.trees_per_set}x{cfg.fusion.sets_fused} "
                                  f"needs {lanes} lanes (> {B200_FORS_MAX_LANES}); keeping the engine's layout",
                                  stacklevel=2)
            kw = {}
            for key in ("fors_trees_per_set", "fors_sets_fused", "fors_relax", "wots_from_tree", "chunk", "streams",
                        "shared_layers", "shared_auto", "fors_cta_levels", "tree_split", "overlap",
                        "fors_small_batch", "tree_small_batch"):
                if key in b:
                    kw[key] = b[key]
            if "variant" in b:
                kw["variant"] = b["variant"]
            else:
                kw["variant"] = {k: 1 if cfg.backends.get(k) == "tuned" else 0 for k in KERNELS}
            engine.set_config(set_id, **kw)

    @classmethod
    def from_engine(cls, engine, base: "TuningConfig | None" = None) -> "TuningConfig":
        cfg = base or cls.default()
        for set_id in PARAMETER_SETS:
            e = engine.config(set_id)
            cfg.sets[set_id].b200 = {
                "fors_trees_per_set": e["fors_trees_per_set"], "fors_sets_fused": e["fors_sets_fused"],
                "fors_relax": e["fors_relax"], "variant": {k: e["variant"][k] for k in KERNELS},
                "wots_from_tree": e["wots_from_tree"], "chunk": e["chunk"], "streams": e["streams"],
                "shared_layers": e["shared_layers"], "shared_auto": e["shared_auto"],
                "fors_cta_levels": e["fors_cta_levels"], "tree_split": e["tree_split"], "overlap": e["overlap"],
                "fors_small_batch": e["fors_small_batch"], "tree_small_batch": e["tree_small_batch"],
            }
            cfg.sets[set_id].backends = {k: "tuned" if e["variant"][k] else "baseline" for k in KERNELS}
        return cfg

    # -- serialization (config.py:105-162) ---------------------------------
    def to_dict(self) -> dict:
        out = {"seme_per_block": self.seme_per_block, "worker_width": self.worker_width, "sets": {}}
        for set_id, cfg in sorted(self.sets.items()):
            f = cfg.fusion
            row = {
                "fusion": {"lanes_per_set": f.lanes_per_set, "sets_fused": f.sets_fused,
                           "trees_per_set": f.trees_per_set, "lane_utilization": f.lane_utilization,
                           "scratch_utilization": f.scratch_utilization, "sync_score": f.sync_score},
                "padding": {"access_bytes": cfg.padding.access_bytes,
                            "banks_per_access": cfg.padding.banks_per_access,
                            "lane_interval": cfg.padding.lane_interval,
                            "rows_per_region": cfg.padding.rows_per_region},
                "backends": dict(cfg.backends),
                "relax": cfg.relax,
            }
            if cfg.b200:
                row["b200"] = cfg.b200
            out["sets"][set_id] = row
        return out

    @classmethod
    def from_dict(cls, data: dict) -> "TuningConfig":
        try:
            sets = {}
            for set_id, raw in data["sets"].items():
                sets[set_id] = SetConfig(
                    fusion=FusionCandidate(**raw["fusion"]), padding=PaddingScheme(**raw["padding"]),
                    backends=dict(raw["backends"]), relax=bool(raw["relax"]), b200=dict(raw.get("b200", {})))
            cfg = cls(seme_per_block=int(data["seme_per_block"]), worker_width=int(data["worker_width"]), sets=sets)
        except (KeyError, TypeError) as exc:
            raise FormatError(f"malformed tuning config: {exc!r}") from exc
        cfg.validate()
        return cfg

    def save(self, path) -> None:
        Path(path).write_text(json.dumps(self.to_dict(), indent=2) + "\n")

    @classmethod
    def load(cls, path) -> "TuningConfig":
        try:
            data = json.loads(Path(path).read_text())
        except json.JSONDecodeError as exc:
            raise FormatError(f"config {path} is not valid JSON: {exc}") from exc
        return cls.from_dict(data)


def resolve_config(path=None) -> TuningConfig:
    path = path or os.environ.get(ENV_CONFIG_PATH)
    if path:
        return TuningConfig.load(path)
    return TuningConfig.default()
