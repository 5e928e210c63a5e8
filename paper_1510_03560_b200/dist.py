"""Multi-GPU stepping: one process per GPU, torch.distributed for plumbing.

The C-ABI does the heavy lifting.  The fused kernel reads neighbour tiles
owned by other ranks directly from their pools over NVLink (CUDA IPC), and
`plbm_gpu_step` on several ranks synchronises them on the device
(include/plbm_gpu.h, "multi-GPU"):

    k_main        fused kernel of this rank's tiles
    rank barrier  flag words in the peers' sync blocks (NVLink stores)
    k_face, k_p5  psi faces for the next step, criterion, local trigger bits
    rank barrier
    k_check_expand  on EVERY rank over the merged trigger bytes and the
                    lowest error key of all ranks (read over NVLink):
                    identical map, placement and EngineError everywhere

so steps are queued ahead with no host collective and no host round trip
per step.  torch.distributed only exchanges the IPC handles once.

`HostMergeStepper` keeps the round-1 protocol (the host merges the trigger
bytes with an all-reduce every step), and `merge_triggers` is its pure
host-side part, exercised on CPU with gloo.
"""
from __future__ import annotations

import threading
from typing import Callable, Optional

import numpy as np


def merge_triggers(local: np.ndarray, all_reduce_max: Callable[[np.ndarray], np.ndarray]) -> np.ndarray:
    """Every slot is owned by exactly one rank and only the owner sets its
    bits, so MAX (or SUM, or OR) over ranks reproduces the single-GPU trigger
    array exactly."""
    return all_reduce_max(np.ascontiguousarray(local, dtype=np.uint8))


def attach_peers(engine, dist) -> None:
    """Exchange the IPC handles of every rank's pools and sync block, map the
    peers', prepare, and barrier (the protocol's set-up, once per run)."""
    world, rank = dist.get_world_size(), dist.get_rank()
    handles = [None] * world
    dist.all_gather_object(handles, engine.ipc_handles())
    for r, h in enumerate(handles):
        if r != rank:
            engine.open_peer(r, h)
    engine.prepare()
    dist.barrier()


class DistStepper:
    """Drives one rank's GpuEngine: plbm_gpu_step with device-side rank
    barriers and expansion (every rank calls step with the same n)."""

    def __init__(self, engine, dist, device: int):
        self.eng, self.dist = engine, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        attach_peers(engine, dist)

    def step(self, n: int = 1) -> None:
        self.eng.step(n)


class HostMergeStepper:
    """The host-merge protocol: step_main, barrier, step_face, all-reduce(MAX)
    of the trigger bytes, step_end with the merged bytes on every rank.

    NCCL (one GPU per rank): both collectives run on the engine's stream.
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
        attach_peers(engine, dist)

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


def step_ranks_threaded(engines, n: int = 1) -> None:
    """Several ranks' engines in ONE process (tests on one GPU): each rank's
    plbm_gpu_step runs on its own host thread (ctypes releases the GIL), the
    ranks meet in the device-side barriers as separate processes would."""
    errors = [None] * len(engines)

    def run(k, e):
        try:
            e.step(n)
        except Exception as ex:  # re-raised on the caller's thread
            errors[k] = ex

    threads = [threading.Thread(target=run, args=(k, e)) for k, e in enumerate(engines)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for ex in errors:
        if ex is not None:
            raise ex


def step_same_process(engines, n: int = 1, merged_override: Optional[np.ndarray] = None) -> None:
    """The host-merge protocol for several ranks' engines in ONE process: the
    merge is a host-side OR of every engine's local trigger bytes."""
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
