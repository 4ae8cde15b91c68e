"""The consistency sampler's chroma gate without a square root
(csrc/ls_aux.cu k_sample): |c - c_q| < 0.05 (energy.py:182-183, np.linalg.norm
= sqrt of the sum of squares) is tested as s <= kGateSq.  sqrt is correctly
rounded and monotone, so that is exact iff kGateSq is the largest double whose
root rounds below 0.05."""
import math
import re
from pathlib import Path

import numpy as np

SRC = Path(__file__).resolve().parents[1] / "paper_1908_01961_b200" / "csrc" / "ls_aux.cu"


def _constant() -> float:
    m = re.search(r"kGateSq\s*=\s*(0x[0-9a-fA-Fp.+-]+);", SRC.read_text())
    assert m, "kGateSq not found"
    return float.fromhex(m.group(1))


def test_gate_constant_is_the_largest_admitted_square():
    t = _constant()
    assert math.sqrt(t) < 0.05
    assert not math.sqrt(math.nextafter(t, 1.0)) < 0.05


def test_gate_constant_matches_norm_on_random_pairs():
    rng = np.random.default_rng(3)
    t = _constant()
    # differences concentrated around the gate, plus exact boundary cases
    d = rng.normal(scale=0.036, size=(200000, 2))
    d = np.concatenate([d, [[0.05, 0.0], [0.0, 0.05], [0.03, 0.04], [-0.03, 0.04]]])
    ref = np.linalg.norm(d, axis=1) < 0.05
    s2 = d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]
    assert np.array_equal(ref, s2 <= t)
