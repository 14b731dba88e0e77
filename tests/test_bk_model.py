"""NEXT-4 host logic without a GPU: the sequential model of the parallel-BK kernel
(scripts/bk_model.py: the same segment schedule -- 1 x 1 .. b x b first segments, pairwise merges
alternating x and y -- and the same growth / augmentation / adoption steps as csrc/bk.cuh, lanes
written as loops) reaches the oracle's max-flow value on tiny volumes (§3.1)."""
import os
import sys

import numpy as np
import pytest

import oracle
from synth import volumes as V

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
import bk_model  # noqa: E402


@pytest.mark.parametrize("seg", [(1, 1), (2, 3), (4, 4)])
def test_bk_model_matches_oracle(seg):
    for seed in range(1000, 1040):
        c, delta = V.tiny_case(seed)
        assert bk_model.solve(c, delta, *seg) == oracle.colgraph_solve(c, delta)["flow"], seed


def test_bk_model_c1():
    c = V.generate("C1")
    assert bk_model.solve(c, 2, 1, 1) == oracle.colgraph_solve(c, 2)["flow"]
