"""Multi-node scaling of the gradient-to-update step.

The reference only models the paper's 32M8G hierarchy analytically
(perf.cpp:83-121): an intra-node ring over the machine's GPUs and an
inter-node ring over machines, combined by max (overlapping channels) or sum,
with part of the exchange hidden behind the last micro-batch's backward. This
module restates that model (same formulas, same validation errors) and adds a
projection of THIS implementation's step onto M machines x G B200s: an
intra-node ring reduce-scatter over NVLink, an inter-node reduce-scatter of
each GPU's 1/G slice over the network, LAMB on the 1/(M G) shard, and the two
all-gathers in reverse — with the per-stage rates measured on one node.
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import InvalidConfig


def ring_comm_time_s(nbytes: float, n_participants: int, bandwidth_bits_per_s: float) -> float:
    """All-reduce time of a ring (perf.cpp:83-95): 2 (n-1)/n * bytes * 8 / bw."""
    if n_participants < 1:
        raise InvalidConfig("ring needs at least one participant")
    if nbytes < 0.0 or not bandwidth_bits_per_s > 0.0:
        raise InvalidConfig("ring_comm_time_s requires nonnegative bytes and positive bandwidth")
    if n_participants == 1:
        return 0.0
    n = float(n_participants)
    return 2.0 * (n - 1.0) / n * nbytes * 8.0 / bandwidth_bits_per_s


@dataclass
class ClusterSpec:
    """perf.hpp:30-46: the "<X>M<Y>G" topology and its channels."""
    machines: int = 1
    gpus_per_machine: int = 1
    throughput_tokens_per_s: float = 0.0   # per-GPU compute rate
    pcie_bandwidth_bits_per_s: float = 64e9  # intra-node channel
    network_bandwidth_bits_per_s: float = 10e9
    param_count: int = 0
    grad_elem_bytes: int = 4

    def world(self) -> int:
        return self.machines * self.gpus_per_machine

    def grad_bytes(self) -> float:
        return float(self.param_count) * float(self.grad_elem_bytes)

    def validate(self) -> None:
        if self.machines < 1 or self.gpus_per_machine < 1:
            raise InvalidConfig("cluster topology must have at least one device")
        if not self.throughput_tokens_per_s > 0.0:
            raise InvalidConfig("per-GPU throughput must be positive")
        if not (self.pcie_bandwidth_bits_per_s > 0.0 and self.network_bandwidth_bits_per_s > 0.0):
            raise InvalidConfig("bandwidths must be positive")
        if self.param_count == 0:
            raise InvalidConfig("param_count must be positive")
        if self.grad_elem_bytes == 0:
            raise InvalidConfig("grad_elem_bytes must be positive")


@dataclass
class PhaseConfig:
    """perf.hpp:48-61."""
    sequence_length: int = 128
    sentences_per_micro: int = 32
    accumulation: int = 1
    epochs: float = 1.0
    tokens_per_epoch: float = 1.0

    def tokens_per_micro(self) -> float:
        return float(self.sequence_length) * float(self.sentences_per_micro)

    def validate(self) -> None:
        if self.sequence_length < 1 or self.sentences_per_micro < 1:
            raise InvalidConfig("phase shape must be positive")
        if self.accumulation < 1:
            raise InvalidConfig("accumulation must be >= 1")
        if not self.epochs > 0.0:
            raise InvalidConfig("epochs must be positive")
        if not self.tokens_per_epoch > 0.0:
            raise InvalidConfig("tokens_per_epoch must be positive")


@dataclass
class IterationModelOptions:
    """perf.hpp:88-97."""
    overlap_fraction: float = 0.5
    backward_share: float = 2.0 / 3.0
    sum_comm: bool = False


def iteration_time(spec: ClusterSpec, phase: PhaseConfig,
                   opt: IterationModelOptions = IterationModelOptions()) -> dict:
    """perf.cpp:97-121: K micro-steps of compute plus the exchange left over
    after hiding overlap_fraction of it behind the last backward."""
    spec.validate()
    phase.validate()
    if not 0.0 <= opt.overlap_fraction <= 1.0:
        raise InvalidConfig("overlap_fraction must lie in [0,1]")
    if not 0.0 <= opt.backward_share <= 1.0:
        raise InvalidConfig("backward_share must lie in [0,1]")
    micro_s = phase.tokens_per_micro() / spec.throughput_tokens_per_s
    t_compute = phase.accumulation * micro_s
    t_pcie = ring_comm_time_s(spec.grad_bytes(), spec.gpus_per_machine, spec.pcie_bandwidth_bits_per_s)
    t_net = ring_comm_time_s(spec.grad_bytes(), spec.machines, spec.network_bandwidth_bits_per_s)
    t_comm = t_pcie + t_net if opt.sum_comm else max(t_pcie, t_net)
    t_bwd = opt.backward_share * micro_s
    exposed = max(0.0, t_comm - opt.overlap_fraction * t_bwd)
    return {"t_compute": t_compute, "t_pcie": t_pcie, "t_net": t_net, "t_comm": t_comm,
            "t_bwd": t_bwd, "exposed_comm": exposed, "total": t_compute + exposed}


# ---------------------------------------------------------------- projection
@dataclass
class B200Rates:
    """Per-GPU rates measured on one B200 node (DESIGN.md §10,
    profiles/r01_notes.md): sustained HBM streaming of the LAMB passes,
    NVLink per direction as the ring hops and the push achieve it, and the
    inter-node network per GPU (one 400 Gb/s NIC per GPU)."""
    hbm_GBs: float = 6100.0
    nvlink_GBs: float = 700.0
    network_GBs: float = 50.0


def project_step_ms(params: int, K: int, machines: int, gpus_per_machine: int,
                    wire_bytes: int = 2, rates: B200Rates = B200Rates()) -> dict:
    """Projected optimizer-step time of the resident-micro path on M x G
    B200s with a two-level reduce-scatter / all-gather (no stage overlap,
    like the measured single-node step): every rank reads its K binary16
    micros once (2K B/param), reduces over NVLink then over the network,
    runs the two LAMB passes on a 1/(M G) shard (36 B/param on one GPU) and
    gathers fp32 weights back over the network and NVLink."""
    if K < 1 or machines < 1 or gpus_per_machine < 1 or params < 1:
        raise InvalidConfig("project_step_ms: positive sizes required")
    P, G, M, E = float(params), gpus_per_machine, machines, float(wire_bytes)
    N = M * G
    hbm = rates.hbm_GBs * 1e9
    t = {}
    t["read_micros"] = 2.0 * K * P / hbm
    t["rs_intra"] = (G - 1) / G * E * P / (rates.nvlink_GBs * 1e9) if G > 1 else 0.0
    t["rs_inter"] = (M - 1) / M * E * P / G / (rates.network_GBs * 1e9) if M > 1 else 0.0
    # one rank: p1r 12 + 12 B beyond the micros, p2 12 B; sharded: phase 1
    # 24 + E B (phase 2's 16 B of HBM run under the NVLink-bound push)
    t["lamb"] = (36.0 if N == 1 else 24.0 + E) * P / N / hbm
    t["ag_inter"] = (M - 1) / M * 4.0 * P / G / (rates.network_GBs * 1e9) if M > 1 else 0.0
    t["ag_intra"] = (G - 1) / G * 4.0 * P / (rates.nvlink_GBs * 1e9) if G > 1 else 0.0
    total = sum(t.values())
    return {"stages_ms": {k: round(v * 1e3, 4) for k, v in t.items()},
            "step_ms": round(total * 1e3, 4),
            "params_per_s": N * P / total, "world": N}
