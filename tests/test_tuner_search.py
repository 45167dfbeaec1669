"""Host logic of the auto-tuner (NEXT #4): the greedy and hill-climbing
strategies over per-layer candidate lists, with a synthetic evaluator (no GPU).  The tuner module
only imports torch lazily (for timing), so these run on the CPU box."""
import importlib.util
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("tuner", os.path.join(ROOT, "paper_2511_19711_b200", "tuner.py"))
tuner = importlib.util.module_from_spec(spec)
sys.modules["tuner"] = tuner
spec.loader.exec_module(tuner)


class FakeEval:
    """error[layer][k], cost[layer][k] tables."""
    def __init__(self, err, cost):
        self.err, self.costs = err, cost

    def error(self, layer, k):
        return self.err[layer.name][k]

    def objective_value(self, layer, k):
        return self.costs[layer.name][k]


def layers(n_cands):
    return [tuner.Layer(name=f"L{i}", op="gelu", rows=1, cols=1, calib=None, calib_rows=1,
                        candidates=[{"k": k} for k in range(nc)]) for i, nc in enumerate(n_cands)]


def test_greedy_walks_each_layer_until_the_threshold():
    L = layers([4, 3])
    ev = FakeEval({"L0": [0, 0.1, 0.2, 5.0], "L1": [0, 0.3, 0.4]}, {"L0": [10, 8, 6, 1], "L1": [9, 5, 2]})
    r = tuner.GreedyTuner(L, ev, threshold=0.61).run()
    # L0: 0 -> 1 (0.1) -> 2 (0.2) -> 3 would be 5.0: rollback; L1: 1 (0.2+0.3=0.5) ok, 2 (0.6) ok
    assert r["state"] == [2, 2]
    assert r["quality_loss"] == pytest.approx(0.6)
    assert r["cost"] == 8 and r["cost_most_accurate"] == 19


def test_greedy_zero_threshold_keeps_the_most_accurate():
    L = layers([3, 3])
    ev = FakeEval({"L0": [0, 0.01, 0.02], "L1": [0, 0.01, 0.5]}, {"L0": [3, 2, 1], "L1": [3, 2, 1]})
    assert tuner.GreedyTuner(L, ev, threshold=0.0).run()["state"] == [0, 0]


def test_greedy_is_order_dependent_hill_climb_takes_the_best_gain():
    # budget 0.5: greedy spends it on L0 (first), hill climbing on L1 (larger cost reduction)
    L = layers([2, 2])
    ev = FakeEval({"L0": [0, 0.5], "L1": [0, 0.5]}, {"L0": [10, 9], "L1": [10, 1]})
    assert tuner.GreedyTuner(L, ev, threshold=0.5).run()["state"] == [1, 0]
    assert tuner.HillClimbTuner(L, ev, threshold=0.5).run()["state"] == [0, 1]


def test_hill_climb_stops_when_no_move_reduces_cost():
    L = layers([3])
    ev = FakeEval({"L0": [0, 0.1, 0.2]}, {"L0": [5, 5, 7]})
    r = tuner.HillClimbTuner(L, ev, threshold=1.0).run()
    assert r["state"] == [0]


def test_network_objective_weights_rounds_and_bytes():
    lat, bw = tuner.NETWORKS["wan"]
    assert lat == pytest.approx(40e-3) and bw == pytest.approx(352e6 / 8)
    lat, bw = tuner.NETWORKS["lan"]
    assert lat == pytest.approx(0.3e-3) and bw == pytest.approx(10e9 / 8)


def test_candidate_lists_start_with_the_most_accurate_knobs():
    c = tuner.CANDIDATES
    assert c["softmax"][0] == dict(exp_t=8, exp_clamp=1)
    assert c["gelu"][-1]["form"] == "relu" and c["layernorm"][0]["rsqrt_iters"] == 3
