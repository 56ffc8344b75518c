"""CPU: the oracle's prefix-sum resamplers (oracle/mgp_oracle.c) against golden vectors of
the unmodified reference (tests/golden/make_golden_prefix.py): np.cumsum order
(M/resample.py:288-291), multinomial (:295-304), systematic_improved (:307-336)."""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
sys.path.insert(0, os.path.dirname(HERE))

from make_golden_prefix import weights_for  # noqa: E402

from oracle import oracle as ora  # noqa: E402

GOLD = json.load(open(os.path.join(HERE, "golden", "golden_prefix.json")))
ARR = np.load(os.path.join(HERE, "golden", "golden_prefix.npz"))
CPU_MAX_N = 1 << 20


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def case_weights(case):
    if "weights" in case:
        return ARR[case["weights"]]
    return weights_for(case["recipe"], lambda y, n, s, p: ora.gen_gaussian_weights(y, n, s, p))


CASES = [c for c in GOLD["cases"] if c["recipe"]["n"] <= CPU_MAX_N]


def test_golden_has_cases():
    assert len(GOLD["cases"]) >= 60
    assert any(c["recipe"]["n"] > (1 << 24) for c in GOLD["cases"])  # the tie-saturation case


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['id']}-{c['recipe']['family']}-{c['recipe']['precision']}-{c['recipe']['n']}")
def test_oracle_prefix_matches_reference(case):
    w = case_weights(case)
    assert sha(w) == case["weights_sha"]
    cum = ora.cumsum(w)
    assert sha(cum) == case["cum_sha"]
    for ent in case["multinomial"]:
        a = ora.multinomial(w, ent["seed"])
        assert sha(a) == ent["sha"], ("multinomial", ent["seed"])
    for ent in case["systematic"]:
        a = ora.systematic(w, ent["seed"])
        assert sha(a) == ent["sha"], ("systematic", ent["seed"])
