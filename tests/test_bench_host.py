"""Host-side pieces of bench.py (no GPU): the algorithmic work per particle behind the
`roofline` objects, counted here by brute-force enumeration, and the clock-sample parser."""
import itertools

import pytest

import bench


def support(order):
    r = range(order + 1)
    return list(itertools.product(r, r, r))


def pair_index(order, i, j):
    # index of the per-axis pair product w_i w_j: unordered pairs for TSC, i + j for CIC
    # (CIC: w0 w1 = w1 w0, and (0,0),(0,1),(1,1) are the distinct products)
    return i + j if order == 1 else sorted([(a, b) for a in range(3) for b in range(a, 3)]).index(tuple(sorted((i, j))))


@pytest.mark.parametrize("order,ncomp", [(1, 9), (2, 9), (1, 1), (2, 1)])
def test_unique_flops_by_enumeration(order, ncomp):
    nodes = support(order)
    pairs = [(a, b) for ai, a in enumerate(nodes) for b in nodes[ai:]]   # unordered node pairs
    assert bench.flops_per_particle(order, ncomp) == 2 * len(pairs) * ncomp


@pytest.mark.parametrize("order,ncomp", [(1, 9), (2, 9), (1, 1), (2, 1)])
def test_pair_product_flops_by_enumeration(order, ncomp):
    nodes = support(order)
    xs = {(pair_index(order, a[0], b[0]), pair_index(order, a[1], b[1])) for a in nodes for b in nodes}
    zs = {pair_index(order, a[2], b[2]) for a in nodes for b in nodes}
    assert bench.flops_per_particle(order, ncomp, "pair") == 2 * len(xs) * len(zs) * ncomp


def test_plan_and_executed_flops():
    # the paper's node-tile plan: 64 (CIC, 8x8 tile) | 640 (TSC, 10 upper 8x8 tiles) MMA entries
    assert bench.flops_per_particle(1, 9, "plan") == 2 * 64 * 9
    assert bench.flops_per_particle(2, 9, "plan") == 2 * 640 * 9
    # executed: DMMA.8x8x4 = 8*8*4 FMA = 512 FLOP per 4 particles; tensor 5 | 35, scalar 2 | 5
    for order, ncomp, ndmma in ((1, 9, 5), (2, 9, 35), (1, 1, 2), (2, 1, 5)):
        assert bench.flops_per_particle(order, ncomp, "executed") == ndmma * 8 * 8 * 4 * 2 // 4


def test_alg_bytes():
    # tensor: x, q, B (7 FP64) in + the node row share S C 8 / ppc out; scalar: x, q (4 FP64)
    assert bench.alg_bytes_per_particle(1, 9, 64) == 56 + 27 * 9 * 8 / 64
    assert bench.alg_bytes_per_particle(2, 9, 64) == 56 + 125 * 9 * 8 / 64
    assert bench.alg_bytes_per_particle(2, 1, 64.25) == 32 + 125 * 8 / 64.25


def test_clock_summary():
    c = bench.ClockSampler(0)
    c.sm, c.mx, c.reasons = [1965.0, 1950.0, 1965.0], 1965.0, {"sw_power_cap"}
    s = c.summary()
    assert s["samples"] == 3 and s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"]
    c.sm = []
    assert c.summary()["samples"] == 0
    # NVML reason bits map to the names the driver checks
    assert set(bench.ClockSampler.REASONS.values()) == {"hw_slowdown", "hw_thermal_slowdown",
                                                        "sw_thermal_slowdown", "sw_power_cap"}
