"""Decision / certificate / output comparison of one head-step, device against
a CPU reference (the oracle restatement or frozen outputs of the unmodified
reference), with the threshold-distance rule of the north star: decisions
must be identical unless a deciding quantity sits within the stated tolerance
of its threshold (oracle/margins.py); numbers are compared whenever the
decisions agree.
"""

import numpy as np

from oracle.margins import FIELDS, near_threshold

KINDS = ("quantized", "dense_per_head", "dense_all_heads")


class Report:
    """Per-run tally of matched decisions and near-threshold exceptions."""

    def __init__(self, name):
        self.name, self.n, self.match, self.exceptions, self.failures = name, 0, 0, [], []
        self.max_err = {}

    def err(self, key, v):
        self.max_err[key] = max(self.max_err.get(key, 0.0), float(v))

    def line(self):
        rate = self.match / self.n if self.n else 1.0
        errs = " ".join(f"{k}={v:.2e}" for k, v in sorted(self.max_err.items()))
        return (f"[parity {self.name}] head-steps={self.n} decisions identical={self.match} "
                f"({100 * rate:.2f}%) near-threshold exceptions={len(self.exceptions)} "
                f"failures={len(self.failures)} max-errors: {errs}")

    def print(self):
        print(self.line())
        for e in self.exceptions[:20]:
            print("   near-threshold:", e)
        for f in self.failures[:20]:
            print("   FAILURE:", f)


def flags_of(bits, lib):
    return (bool(bits & lib.F_RUNG1), bool(bits & lib.F_RUNG2),
            bool(bits & (lib.F_RANKING | lib.F_BOUNDARY)),
            bool(bits & (lib.F_CANARY | lib.F_NUMERIC | lib.F_EXPLORE)))


def compare(rep, ctx, dev, ref, margins, tol, num_tol):
    """dev / ref: dicts with promoted, vprom (sorted lists), k_star, flags (4
    bools), kind (str), delta_h, e_key_tight, e_key_impl, e_val, est_tail_mass,
    output (ndarray).  ``num_tol``: rel tolerances {key: rtol} plus
    'out_quant' / 'out_dense' (relative to max|O|)."""
    rep.n += 1
    same = (dev["promoted"] == ref["promoted"] and dev["vprom"] == ref["vprom"]
            and dev["k_star"] == ref["k_star"] and tuple(dev["flags"]) == tuple(ref["flags"])
            and dev["kind"] == ref["kind"])
    if not same:
        near = near_threshold(margins, tol)
        what = {k: (dev[k], ref[k]) for k in ("k_star", "flags", "kind") if dev[k] != ref[k]}
        if dev["promoted"] != ref["promoted"]:
            what["promoted_diff"] = sorted(set(dev["promoted"]) ^ set(ref["promoted"]))[:8]
        if dev["vprom"] != ref["vprom"]:
            what["vprom_diff"] = sorted(set(dev["vprom"]) ^ set(ref["vprom"]))[:8]
        info = f"{ctx}: {what} margins={{{', '.join(f'{k}: {margins[k]:.2e}' for k in FIELDS)}}}"
        if near:
            rep.exceptions.append(info + f" near={near}")
        else:
            rep.failures.append(info)
        return
    rep.match += 1
    for key in ("delta_h", "e_key_tight", "e_key_impl", "e_val", "est_tail_mass"):
        a, b = float(dev[key]), float(ref[key])
        err = abs(a - b) / max(abs(b), 1e-12) if abs(b) > 1e-9 else abs(a - b)
        rep.err(key, err)
        if err > num_tol[key]:
            rep.failures.append(f"{ctx}: {key} {a!r} vs {b!r} (rel {err:.2e})")
    o_d, o_r = np.asarray(dev["output"], np.float64), np.asarray(ref["output"], np.float64)
    # relative to max|O|, or to the RMS of the unit's values when given: at long
    # context O averages ~N values and is far smaller than they are, while fp32
    # accumulation error scales with the values
    scale = max(np.abs(o_r).max(), float(ref.get("vscale", 0.0)), 1e-30)
    err = np.abs(o_d - o_r).max() / scale
    key = "out_quant" if ref["kind"] == "quantized" else "out_dense"
    rep.err(key, err)
    if err > num_tol[key]:
        rep.failures.append(f"{ctx}: output ({ref['kind']}) rel err {err:.2e}")


def dev_row(cert_row, kind, promoted, vprom, output, lib):
    return {"promoted": sorted(int(b) for b in promoted), "vprom": sorted(int(b) for b in vprom),
            "k_star": int(cert_row["k_star"]), "flags": flags_of(int(cert_row["flags"]), lib),
            "kind": KINDS[int(kind)], "delta_h": cert_row["delta_h"],
            "e_key_tight": cert_row["e_key_tight"], "e_key_impl": cert_row["e_key_impl"],
            "e_val": cert_row["e_val"], "est_tail_mass": cert_row["est_tail_mass"],
            "output": output}


def oracle_row(r, kind=None, output=None):
    return {"promoted": [int(b) for b in r["promoted"]],
            "vprom": [int(b) for b in r["value_promotions"]], "k_star": int(r["k_star"]),
            "flags": tuple(bool(x) for x in r["flags"]), "kind": kind or r["kind"],
            "delta_h": r["delta_h"], "e_key_tight": r["e_key_tight"],
            "e_key_impl": r["e_key_impl"], "e_val": r["e_val"],
            "est_tail_mass": r["est_tail_mass"],
            "output": r["output"] if output is None else output}


def log(rep):
    """Print the report; with CKV_PARITY_LOG set also append it to that file
    (the GPU runs collect the per-config match rates there)."""
    import os
    rep.print()
    path = os.environ.get("CKV_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(rep.line() + "\n")
            for e in rep.exceptions[:50]:
                f.write("   near-threshold: " + e + "\n")
            for e in rep.failures[:50]:
                f.write("   FAILURE: " + e + "\n")
