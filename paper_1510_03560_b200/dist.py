"""Multi-GPU stepping: one process per GPU, torch.distributed for plumbing.

The C-ABI does the heavy lifting (the fused kernel reads neighbour tiles owned
by other ranks directly from their pools over NVLink, CUDA IPC); this module
is the per-step protocol between ranks (include/plbm_gpu.h "multi-GPU"):

    step_main    fused kernel of this rank's tiles
    barrier      k_face pulls peers' freshly written f_post (1-element
                 all-reduce on the engine stream)
    step_face    psi faces for the next step, criterion, local trigger bits
    all-reduce   MAX over ranks of the trigger bytes (stream-ordered NCCL;
                 also orders the double-buffered pools for the next step)
    step_end     identical expansion / placement on every rank's mirror

`merge_triggers` is the pure host-side part, exercised on CPU with gloo.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np


def merge_triggers(local: np.ndarray, all_reduce_max: Callable[[np.ndarray], np.ndarray]) -> np.ndarray:
    """Every slot is owned by exactly one rank and only the owner sets its
    bits, so MAX (or SUM, or OR) over ranks reproduces the single-GPU trigger
    array exactly."""
    return all_reduce_max(np.ascontiguousarray(local, dtype=np.uint8))


class DistStepper:
    """Drives one rank's GpuEngine with torch.distributed.

    NCCL (one GPU per rank): both collectives run on the engine's stream, so
    the host never waits for the kernels except to read the merged triggers.
    gloo (tests: several ranks sharing one GPU): the engine stream is synced
    and the collectives run on host tensors."""

    def __init__(self, engine, dist, device: int):
        import torch
        self.eng, self.dist, self.torch = engine, dist, torch
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.nccl = dist.get_backend() == "nccl"
        self.stream = torch.cuda.ExternalStream(engine.stream(), device=torch.device("cuda", device))
        n = engine.trigger_bytes()
        dev = f"cuda:{device}" if self.nccl else "cpu"
        self.trig = torch.empty(n, dtype=torch.uint8, device=dev)
        self.token = torch.zeros(1, dtype=torch.int32, device=dev)
        self._attach_peers()

    def _attach_peers(self) -> None:
        handles = [None] * self.world
        self.dist.all_gather_object(handles, self.eng.ipc_handles())
        for r, h in enumerate(handles):
            if r != self.rank:
                self.eng.open_peer(r, h)
        self.eng.prepare()
        self.dist.barrier()

    def step(self, n: int = 1) -> None:
        torch = self.torch
        if not self.nccl:
            for _ in range(n):
                self.eng.step_main()
                self.eng.sync()
                self.dist.all_reduce(self.token)  # barrier: peers' f_post^(k) complete
                self.eng.step_face()
                local = self.eng.local_triggers()
                t = torch.from_numpy(local)
                self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
                self.eng.step_end(t.numpy())
            return
        with torch.cuda.stream(self.stream):
            for _ in range(n):
                self.eng.step_main()
                self.dist.all_reduce(self.token)  # barrier: peers' f_post^(k) complete
                self.eng.step_face()
                src = _device_u8(self.eng.triggers_device(), self.trig.numel(), self.trig.device)
                self.trig.copy_(src)
                self.dist.all_reduce(self.trig, op=self.dist.ReduceOp.MAX)
                merged = self.trig.cpu().numpy()
                self.eng.step_end(merged)


def _device_u8(ptr: int, n: int, device) -> "torch.Tensor":
    """Zero-copy torch view of a device byte array owned by the engine."""
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3}
    return torch.as_tensor(_CAI(), device=device)


def step_same_process(engines, n: int = 1, merged_override: Optional[np.ndarray] = None) -> None:
    """Several ranks' engines in ONE process (tests on one GPU): the merge is
    a host-side OR of every engine's local trigger bytes."""
    for _ in range(n):
        for e in engines:
            e.step_main()
        for e in engines:
            e.sync()
        for e in engines:
            e.step_face()
        for e in engines:
            e.sync()
        merged = np.zeros(engines[0].trigger_bytes(), np.uint8)
        for e in engines:
            merged |= e.local_triggers()
        for e in engines:
            e.step_end(merged if merged_override is None else merged_override)
