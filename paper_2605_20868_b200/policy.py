"""Certificate policy, fallback events and certificates (host-side types).

Same names, fields, defaults and validation as the reference
(fallback.py:23-131, certifier.py:20-86) so code written against ``certkv``
keeps working; the device copy of the policy is ``PolicyConfig.to_c()``.
"""

import dataclasses
from dataclasses import dataclass, field

from . import _lib

CAUSE_COVERAGE = "coverage_expand"
CAUSE_VALUE_TOL = "value_tol"
CAUSE_RANKING = "ranking_disagree"
CAUSE_BOUNDARY = "boundary"
CAUSE_CANARY = "canary"
CAUSE_PRECONDITION = "precondition"
CAUSES = frozenset({CAUSE_COVERAGE, CAUSE_VALUE_TOL, CAUSE_RANKING, CAUSE_BOUNDARY,
                    CAUSE_CANARY, CAUSE_PRECONDITION})
RUNG4_CAUSES = frozenset({CAUSE_CANARY, CAUSE_PRECONDITION})

RETURNED_QUANTIZED = "quantized"
RETURNED_DENSE_PER_HEAD = "dense_per_head"
RETURNED_DENSE_ALL_HEADS = "dense_all_heads"
KINDS = (RETURNED_QUANTIZED, RETURNED_DENSE_PER_HEAD, RETURNED_DENSE_ALL_HEADS)


@dataclass(frozen=True)
class PolicyConfig:
    """Runtime certificate policy (fallback.py:35-111)."""

    tau_cov: float = 0.995
    k_min: int = 2
    k_max: int = 128
    v_tol: float = 0.05
    ranking_depth: int = 1
    epsilon_guard: float = 1e-6
    exploration_rate: float = 0.02
    exponent_mode: int = 3
    greedy_value_budget: float | None = None
    rung1_enabled: bool = True
    rung2_enabled: bool = True
    ranking_checks_enabled: bool = True
    canary_enabled: bool = True

    def __post_init__(self):
        checks = [
            (0.0 <= self.tau_cov <= 1.0, "tau_cov must be in [0, 1]"),
            (0 <= self.k_min <= self.k_max, "need 0 <= k_min <= k_max"),
            (self.v_tol > 0, "v_tol must be positive"),
            (self.ranking_depth >= 1, "ranking_depth must be at least 1"),
            (self.epsilon_guard >= 0, "epsilon_guard must be non-negative"),
            (self.exploration_rate == 0.0 or 0.01 <= self.exploration_rate <= 0.05,
             "exploration_rate must be 0 or in [0.01, 0.05]"),
            (self.exponent_mode in (2, 3), "exponent_mode must be 2 or 3"),
            (self.greedy_value_budget is None or self.greedy_value_budget >= 0,
             "greedy_value_budget must be non-negative"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)

    @classmethod
    def naive(cls):
        """Certification off: the contrast configuration (fallback.py:79-87)."""
        return cls(k_min=0, k_max=0, exploration_rate=0.0, rung1_enabled=False,
                   rung2_enabled=False, ranking_checks_enabled=False, canary_enabled=False)

    def to_dict(self):
        return {f.name: getattr(self, f.name) for f in dataclasses.fields(self)}

    @classmethod
    def from_dict(cls, data):
        unknown = set(data) - {f.name for f in dataclasses.fields(cls)}
        if unknown:
            raise ValueError(f"unknown policy fields: {sorted(unknown)}")
        return cls(**data)

    def to_c(self):
        return _lib.CkvPolicy(
            tau_cov=self.tau_cov, v_tol=self.v_tol, epsilon_guard=self.epsilon_guard,
            greedy_value_budget=-1.0 if self.greedy_value_budget is None else self.greedy_value_budget,
            k_min=self.k_min, k_max=self.k_max, ranking_depth=self.ranking_depth,
            exponent_mode=self.exponent_mode, rung1_enabled=int(self.rung1_enabled),
            rung2_enabled=int(self.rung2_enabled),
            ranking_checks_enabled=int(self.ranking_checks_enabled),
            canary_enabled=int(self.canary_enabled))


@dataclass(frozen=True)
class FallbackEvent:
    """One rung firing for one head in one step (fallback.py:114-131)."""

    rung: int
    head: int
    step: int
    cause: str

    def __post_init__(self):
        if self.cause not in CAUSES:
            raise ValueError(f"unknown cause {self.cause!r}")
        if self.rung not in (1, 2, 3, 4):
            raise ValueError(f"rung must be 1..4, got {self.rung}")
        if self.rung == 4 and self.cause not in RUNG4_CAUSES:
            raise ValueError("rung 4 events are canary or precondition only")

    def to_dict(self):
        return {"rung": self.rung, "head": self.head, "step": self.step, "cause": self.cause}


@dataclass(frozen=True)
class RungFlags:
    rung1: bool = False
    rung2: bool = False
    rung3: bool = False
    rung4: bool = False

    def to_dict(self):
        return {"rung1": self.rung1, "rung2": self.rung2, "rung3": self.rung3, "rung4": self.rung4}


@dataclass(frozen=True)
class Certificate:
    """Per-head per-step bounds and the returned output kind (certifier.py:36-86)."""

    head: int
    step: int
    delta_h: float
    e_key_tight: float
    e_key_impl: float
    e_val: float
    est_tail_mass: float
    v_max: float
    k_star: int
    returned_kind: str
    rung_flags: RungFlags = field(default_factory=RungFlags)

    @property
    def is_dense(self):
        return self.returned_kind != RETURNED_QUANTIZED

    @property
    def returned_e_key(self):
        return 0.0 if self.is_dense else self.e_key_impl

    @property
    def returned_e_val(self):
        return 0.0 if self.is_dense else self.e_val

    def to_dict(self):
        return {"head": self.head, "step": self.step, "delta_h": self.delta_h,
                "e_key_tight": self.e_key_tight, "e_key_impl": self.e_key_impl,
                "e_val": self.e_val, "est_tail_mass": self.est_tail_mass,
                "v_max": self.v_max, "k_star": self.k_star,
                "returned_kind": self.returned_kind,
                "returned_e_key": self.returned_e_key,
                "returned_e_val": self.returned_e_val,
                "rung_flags": self.rung_flags.to_dict()}


def events_from_flags(flags, head, step):
    """Device flag word -> FallbackEvent list in the reference's emission order
    (harness.py:202-269: rung1, rung2, ranking, boundary, canary)."""
    ev = []
    if flags & _lib.F_RUNG1:
        ev.append(FallbackEvent(1, head, step, CAUSE_COVERAGE))
    if flags & _lib.F_RUNG2:
        ev.append(FallbackEvent(2, head, step, CAUSE_VALUE_TOL))
    if flags & _lib.F_RANKING:
        ev.append(FallbackEvent(3, head, step, CAUSE_RANKING))
    if flags & _lib.F_BOUNDARY:
        ev.append(FallbackEvent(3, head, step, CAUSE_BOUNDARY))
    if flags & _lib.F_CANARY:
        ev.append(FallbackEvent(4, head, step, CAUSE_CANARY))
    if flags & _lib.F_EXPLORE:
        ev.append(FallbackEvent(4, head, step, CAUSE_CANARY))
    if flags & _lib.F_NUMERIC:
        ev.append(FallbackEvent(4, head, step, CAUSE_PRECONDITION))
    return ev


def e_key_bound(v_max, delta, est_tail_mass, exponent_mode):
    """E_key = 2 v_max e^{e Delta} alpha_T (e^{2 Delta} - 1), e in {2, 3}
    (certifier.py:135-144) -- the formula k_combine evaluates in fp64."""
    if exponent_mode not in (2, 3):
        raise ValueError("exponent_mode must be 2 or 3")
    import math
    return (2.0 * float(v_max) * math.exp(exponent_mode * float(delta)) * float(est_tail_mass)
            * (math.exp(2.0 * float(delta)) - 1.0))
