"""Chained execution of prepacked QNN layers (the "fused operator" sequence the
paper's compiler would emit, fig:overview P:197-213) with device-resident
buffers and CUDA-graph replay.

A stack is built from layer specs plus weight tensors that the caller owns
(synthetic in the bench); every launch goes through the C ABI.  Glue ops that
are not on this hot path (max pool, residual add, global average pool) are
not executed: a layer whose producer is not a conv reads a persistent buffer
of the right shape ("Workloads").
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import qnn


@dataclass
class LayerSpec:
    name: str
    N: int
    H: int
    W: int
    C: int
    K: int
    R: int
    S: int
    stride: tuple
    pad: tuple
    groups: int
    zp_A: int
    s_A: float
    zp_W: int
    s_W: object          # list / array of 1 or K floats
    out: dict            # requantize params (scale, zero_point, dtype, rounding, relu, act_min, act_max)
    src: str             # producer layer name or "" for a persistent input buffer
    input_dtype: str = "u8"

    @property
    def P(self):
        return (self.H + self.pad[0] + self.pad[2] - self.R) // self.stride[0] + 1

    @property
    def Q(self):
        return (self.W + self.pad[1] + self.pad[3] - self.S) // self.stride[1] + 1

    def macs(self):
        return self.N * self.P * self.Q * self.K * (self.C // self.groups) * self.R * self.S


class ConvStack:
    """Prepacked conv layers + activation buffers on one device."""

    def __init__(self, specs: list[LayerSpec], weights: dict, biases: dict, fresh_inputs: dict, device):
        self.specs = specs
        self.device = device
        self.ops = {}
        self.outs = {}
        self.inputs = {}
        for sp in specs:
            op = qnn.PackedConv2d(sp.N, sp.H, sp.W, sp.C, weights[sp.name], biases.get(sp.name), sp.zp_A, sp.zp_W,
                                  sp.s_A, sp.s_W, sp.out, sp.stride, sp.pad, (1, 1), sp.groups,
                                  input_dtype=sp.input_dtype)
            self.ops[sp.name] = op
            self.outs[sp.name] = torch.empty(op.out_shape(), dtype=op.out_dtype, device=device)
        for sp in specs:
            if sp.src:
                self.inputs[sp.name] = self.outs[sp.src]
            else:
                self.inputs[sp.name] = fresh_inputs[sp.name]

    def run(self, stream=None, events=None):
        """Enqueue every layer; optional per-layer (start, end) CUDA events for timing."""
        for i, sp in enumerate(self.specs):
            if events is not None:
                events[i][0].record()
            self.ops[sp.name](self.inputs[sp.name], out=self.outs[sp.name], stream=stream)
            if events is not None:
                events[i][1].record()

    def total_macs(self):
        return sum(sp.macs() for sp in self.specs)
