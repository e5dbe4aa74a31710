"""the reference's analytic multi-node model
(perf.cpp:83-121), restated, checked against the reference's own tests
(test_perf.cpp:158-181, 222-281), plus the B200 projection's consistency with
the measured single-node steps."""
import math

import pytest

from paper_2008_00177_b200.errors import InvalidConfig
from paper_2008_00177_b200.scaling import (ClusterSpec, IterationModelOptions, PhaseConfig,
                                           iteration_time, project_step_ms, ring_comm_time_s)


def t4_cluster(machines, gpus, throughput=5429.1):
    return ClusterSpec(machines, gpus, throughput, 64e9, 10e9, 340000000, 4)


def phase1(accumulation=1):
    return PhaseConfig(128, 32, accumulation, 36.0, 16752.7e6)


def test_ring_closed_form():
    gib = 1073741824.0
    t = ring_comm_time_s(gib, 2, 10e9)
    assert t == pytest.approx(2.0 * 0.5 * gib * 8.0 / 10e9)
    assert t == pytest.approx(0.859, rel=1e-3)
    assert ring_comm_time_s(gib, 1, 10e9) == 0.0
    assert ring_comm_time_s(0.0, 8, 10e9) == 0.0
    asymptote = 2.0 * gib * 8.0 / 10e9
    prev, n = 0.0, 2
    while n <= 4096:
        cur = ring_comm_time_s(gib, n, 10e9)
        assert prev < cur < asymptote
        prev, n = cur, n * 2
    assert prev > 0.999 * asymptote
    for args in [(gib, 0, 10e9), (-1.0, 2, 10e9), (gib, 2, 0.0)]:
        with pytest.raises(InvalidConfig):
            ring_comm_time_s(*args)


def test_iteration_time_limit_cases():
    b = iteration_time(t4_cluster(1, 1), phase1(1), IterationModelOptions(overlap_fraction=0.0))
    assert b["t_pcie"] == 0.0 and b["t_net"] == 0.0 and b["t_comm"] == 0.0
    assert b["total"] == b["t_compute"]
    assert b["t_compute"] == pytest.approx(4096.0 / 5429.1)
    c = t4_cluster(1, 2)
    c.param_count = 1000000
    b = iteration_time(c, phase1(1), IterationModelOptions(overlap_fraction=1.0))
    assert 0.0 < b["t_comm"] <= b["t_bwd"] and b["exposed_comm"] == 0.0
    assert b["total"] == b["t_compute"]
    b = iteration_time(t4_cluster(2, 1), phase1(1))
    assert b["t_comm"] >= b["t_compute"]
    c = t4_cluster(4, 4)
    bmax = iteration_time(c, phase1(1))
    bsum = iteration_time(c, phase1(1), IterationModelOptions(sum_comm=True))
    assert bsum["t_comm"] == pytest.approx(bsum["t_pcie"] + bsum["t_net"])
    assert bmax["t_comm"] == pytest.approx(max(bmax["t_pcie"], bmax["t_net"]))
    assert bsum["t_comm"] > bmax["t_comm"] and bsum["total"] >= bmax["total"]
    with pytest.raises(InvalidConfig):
        iteration_time(t4_cluster(1, 1), phase1(1), IterationModelOptions(overlap_fraction=1.5))
    with pytest.raises(InvalidConfig):
        iteration_time(t4_cluster(1, 1), phase1(1), IterationModelOptions(backward_share=-0.1))
    bad = t4_cluster(1, 1)
    bad.param_count = 0
    with pytest.raises(InvalidConfig):
        iteration_time(bad, phase1(1))
    with pytest.raises(InvalidConfig):
        iteration_time(t4_cluster(1, 1), phase1(0))


def test_b200_projection_tracks_single_node_measurements():
    """Within 10% of the measured steps of the stage-serial path the model
    describes (2.28 / 2.51 / 2.85 ms at 1 / 2 / 4 GPUs; the
    grouped LAMB default at 4 GPUs, 2.60 ms, overlaps stages the model adds)."""
    P = 336226108
    for g, measured in [(1, 2.28), (2, 2.51), (4, 2.85)]:
        proj = project_step_ms(P, 4, 1, g)
        assert math.isclose(proj["step_ms"], measured, rel_tol=0.10), (g, proj)
    # more machines add the network stages; the step never gets shorter
    one = project_step_ms(P, 4, 1, 8)["step_ms"]
    many = project_step_ms(P, 4, 32, 8)
    assert many["step_ms"] > one and many["world"] == 256
