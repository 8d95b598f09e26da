"""The reference's verification suites (verification.py:61-611) through the
package's device-backed ``verification`` module.  Host-only lemmas run on CPU;
the properties of the device path (reconstruction, value error, output
soundness, fallback exactness, ranking certificate) run on the B200 at reduced
trial counts."""

import os

import pytest

from paper_2605_20868_b200 import verification as V


@pytest.mark.parametrize("name", ["softmax_perturbation", "mass_estimation", "paper_constants",
                                  "storage_accounting", "gqa_union"])
def test_host_lemmas(name):
    fn = V.RUNNERS[name]
    r = fn(trials=20_000) if name in V.DEFAULT_TRIALS else fn()
    print(r.line())
    assert r.ok, r.line()


def test_registry_matches_reference():
    assert V.SUITES == {
        "bounds": ("reconstruction_bounds", "value_error_bound", "softmax_perturbation",
                   "mass_estimation", "output_soundness", "paper_constants"),
        "fallback": ("fallback_exactness", "ranking_certificate"),
        "storage": ("storage_accounting", "gqa_union")}
    with pytest.raises(ValueError, match="unknown suite"):
        V.run_suite("nope")


DEVICE = [("reconstruction_bounds", 20_000), ("value_error_bound", 4_000),
          ("output_soundness", 600), ("fallback_exactness", 150), ("ranking_certificate", 600)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,trials", DEVICE, ids=[d[0] for d in DEVICE])
def test_device_property(name, trials):
    import __graft_entry__
    __graft_entry__.build()
    r = V.RUNNERS[name](trials=trials, seed=0)
    print(r.line())
    path = os.environ.get("CKV_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write("[verify] " + r.line() + "\n")
    assert r.ok, r.line()
