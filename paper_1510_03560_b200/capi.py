"""ctypes bindings for the step-loop C-ABI.

Three libraries export the same surface with different prefixes:

  plbm_gpu_*     libplbm_gpu.so   — the product (B200 engine, include/plbm_gpu.h)
  plbm_oracle_*  oracle/_build/libplbm_oracle.so — C restatement (tests only)
  plbm_ref_*     oracle/_ref/libplbm_ref.so      — the reference itself (tests only)

This module only binds symbols; it never falls back from one library to
another.  A missing product library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Tuple

import numpy as np

from .scenario import (Counters, CreationEvent, EngineError, Error, FACE_NAMES,
                       FIELD_F, Scenario)

_HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(_HERE)
GPU_LIB = os.environ.get("PLBM_GPU_LIB", os.path.join(_HERE, "libplbm_gpu.so"))
ORACLE_LIB = os.path.join(REPO, "oracle", "_build", "libplbm_oracle.so")
REF_LIB = os.path.join(REPO, "oracle", "_ref", "libplbm_ref.so")

_libs: Dict[str, C.CDLL] = {}


def _bind(lib: C.CDLL, prefix: str) -> None:
    P = C.c_void_p
    i32p = C.POINTER(C.c_int32)
    f = lambda n: getattr(lib, f"{prefix}_{n}")  # noqa: E731
    f("create").restype = P
    f("create").argtypes = [P, C.c_int, C.POINTER(Error)]
    f("step").restype = C.c_int
    f("step").argtypes = [P, C.c_int, C.POINTER(Error)]
    f("counters").restype = None
    f("counters").argtypes = [P, C.POINTER(Counters)]
    f("tiles").restype = C.c_int
    f("tiles").argtypes = [P, i32p, i32p, C.POINTER(C.c_int64), C.c_int]
    f("read_tile").restype = C.c_int
    f("read_tile").argtypes = [P, i32p, C.c_int, C.c_int, C.POINTER(C.c_double)]
    f("creation_log").restype = C.c_int
    f("creation_log").argtypes = [P, C.POINTER(CreationEvent), C.c_int]
    f("poke_f").restype = C.c_int
    f("poke_f").argtypes = [P, i32p, C.c_int, C.c_int, i32p, C.c_double]
    f("destroy").restype = None
    f("destroy").argtypes = [P]


def load(path: str, prefix: str) -> C.CDLL:
    key = f"{path}:{prefix}"
    if key not in _libs:
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} is not built — run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(path)
        _bind(lib, prefix)
        _libs[key] = lib
    return _libs[key]


class StepEngine:
    """One engine instance behind the C-ABI (Engine's shape:
    proj/include/plbm/engine.hpp:98-116)."""

    def __init__(self, scenario: Scenario, lib_path: str, prefix: str, workers: int = 0):
        self.scenario = scenario
        self.prefix = prefix
        self.lib = load(lib_path, prefix)
        self._c = scenario.to_c()
        err = Error()
        self._h = self._fn("create")(C.cast(self._c.ptr(), C.c_void_p), workers, C.byref(err))
        if not self._h:
            raise ValueError(f"{prefix}_create failed: {err.message.decode()}")
        E = scenario.tile_extent
        self.ncell = E ** 3

    def _fn(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    def step(self, n: int = 1) -> None:
        err = Error()
        rc = self._fn("step")(self._h, n, C.byref(err))
        if rc != 0:
            raise EngineError(err)

    def counters(self) -> dict:
        c = Counters()
        self._fn("counters")(self._h, C.byref(c))
        return c.as_dict()

    def tiles(self) -> List[Tuple[Tuple[int, int, int], int, int]]:
        n = self._fn("tiles")(self._h, None, None, None, 0)
        coords = (C.c_int32 * (3 * max(n, 1)))()
        owners = (C.c_int32 * max(n, 1))()
        births = (C.c_int64 * max(n, 1))()
        self._fn("tiles")(self._h, coords, owners, births, n)
        return [((coords[3 * k], coords[3 * k + 1], coords[3 * k + 2]), owners[k], births[k])
                for k in range(n)]

    def read_tile(self, coords, comp: int, fld: int) -> np.ndarray:
        E = self.scenario.tile_extent
        n = self.ncell * (19 if fld == FIELD_F else 1)
        out = np.empty(n, dtype=np.float64)
        cc = (C.c_int32 * 3)(*coords)
        rc = self._fn("read_tile")(self._h, cc, comp, fld,
                                   out.ctypes.data_as(C.POINTER(C.c_double)))
        if rc != 0:
            raise KeyError(f"read_tile{tuple(coords)} comp {comp} field {fld}: rc={rc}")
        if fld == FIELD_F:
            return out.reshape(19, E, E, E)
        return out.reshape(E, E, E)

    def creation_log(self) -> List[Tuple[int, Tuple[int, int, int], str, int]]:
        n = self._fn("creation_log")(self._h, None, 0)
        buf = (CreationEvent * max(n, 1))()
        self._fn("creation_log")(self._h, buf, n)
        return [(buf[k].iteration, tuple(buf[k].coords),
                 "init" if buf[k].trigger < 0 else FACE_NAMES[buf[k].trigger], buf[k].owner)
                for k in range(n)]

    def poke_f(self, coords, comp: int, i: int, local, value: float) -> None:
        cc = (C.c_int32 * 3)(*coords)
        ll = (C.c_int32 * 3)(*local)
        if self._fn("poke_f")(self._h, cc, comp, i, ll, value) != 0:
            raise KeyError("poke_f: no such tile")

    def dump_field(self, field: str, comp: int, iteration: int, base_path: str,
                   with_pgm: bool = False) -> None:
        """iobench::dump_field (proj/src/dump.cpp:59-125): <base>.raw/.meta[/.pgm]."""
        fn = self._fn("dump_field")
        fn.restype = C.c_int
        fn.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_long, C.c_char_p, C.c_int]
        rc = fn(self._h, field.encode(), comp, iteration, base_path.encode(), int(with_pgm))
        if rc != 0:
            raise RuntimeError(f"{self.prefix}_dump_field({field}, {comp}) failed: rc={rc}")

    def close(self) -> None:
        if self._h:
            self._fn("destroy")(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def ref_engine(sc: Scenario, workers: int = 1) -> StepEngine:
    return StepEngine(sc, REF_LIB, "plbm_ref", workers)


def ref_run_scenario(sc: Scenario, output_dir: str, iterations: int, report_interval: int = 10,
                     snapshot_interval: int = 0, fields=("rho",), with_pgm: bool = False,
                     name: str = "shim", workers: int = 1) -> None:
    """The reference driver itself (engine::run_scenario, proj/src/engine.cpp:
    580-704), through the test shim: writes the reference's output files."""
    lib = load(REF_LIB, "plbm_ref")
    fn = lib.plbm_ref_run_scenario
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_int, C.c_long, C.c_int, C.c_int, C.c_char_p, C.c_int,
                   C.c_char_p, C.c_char_p]
    cs = sc.to_c()
    rc = fn(C.cast(cs.ptr(), C.c_void_p), workers, iterations, report_interval, snapshot_interval,
            ",".join(fields).encode(), int(with_pgm), name.encode(), output_dir.encode())
    if rc != 0:
        raise RuntimeError(f"plbm_ref_run_scenario failed: rc={rc}")


def oracle_engine(sc: Scenario) -> StepEngine:
    return StepEngine(sc, ORACLE_LIB, "plbm_oracle", 1)


class KernelStats(C.Structure):
    _fields_ = [("main_launches", C.c_int64), ("main_ms", C.c_double),
                ("face_launches", C.c_int64), ("face_ms", C.c_double),
                ("kernels_launched", C.c_int64), ("main_cell_updates", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64)]


class Options(C.Structure):
    """plbm_gpu_options (include/plbm_gpu.h)."""
    _fields_ = [("storage", C.c_int32), ("reserved", C.c_int32 * 7)]


STORAGE = {"ab": 0, "aa": 1}  # PLBM_STORAGE_AB / PLBM_STORAGE_AA


class GpuEngine(StepEngine):
    """The product engine (libplbm_gpu.so).  There is no fallback: a missing
    library or CUDA device raises.  rank/world > 1 builds one rank of a
    multi-GPU run (include/plbm_gpu.h, "multi-GPU")."""

    def __init__(self, sc: Scenario, device: int = 0, capture: bool = False,
                 rank: int = 0, world: int = 1, storage: str = "ab"):
        if storage not in STORAGE:
            raise ValueError(f"storage must be one of {sorted(STORAGE)}")
        self.rank, self.world, self.storage = rank, world, storage
        self.scenario, self.prefix = sc, "plbm_gpu"
        self.lib = load(GPU_LIB, "plbm_gpu")
        self.lib.plbm_gpu_create_ex.restype = C.c_void_p
        self.lib.plbm_gpu_create_ex.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int,
                                                C.POINTER(Options), C.POINTER(Error)]
        self._c = sc.to_c()
        err = Error()
        opt = Options(storage=STORAGE[storage])
        self._h = self.lib.plbm_gpu_create_ex(C.cast(self._c.ptr(), C.c_void_p), device, rank, world,
                                              C.byref(opt), C.byref(err))
        if not self._h:
            raise ValueError(f"plbm_gpu_create_ex failed: {err.message.decode()}")
        self.ncell = sc.tile_extent ** 3
        lib = self.lib
        P = C.c_void_p
        for name, res, args in [
                ("prepare", C.c_int, [P]),
                ("step_begin", C.c_int, [P, C.POINTER(Error)]),
                ("step_main", C.c_int, [P, C.POINTER(Error)]),
                ("step_face", C.c_int, [P]),
                ("step_end", C.c_int, [P, C.c_void_p, C.POINTER(Error)]),
                ("trigger_bytes", C.c_int, [P]),
                ("triggers_device", C.c_void_p, [P]),
                ("local_triggers", C.c_int, [P, C.c_void_p, C.c_int]),
                ("ipc_handles", C.c_int, [P, C.c_void_p]),
                ("open_peer", C.c_int, [P, C.c_int, C.c_void_p]),
                ("set_peer_pools", C.c_int, [P, C.c_int, C.c_void_p, C.c_void_p]),
                ("pool_pointers", None, [P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
                ("sync_block", C.c_void_p, [P]),
                ("set_peer_sync", C.c_int, [P, C.c_int, C.c_void_p]),
                ("tile_rank", C.c_int, [P, C.POINTER(C.c_int32)]),
                ("sync", C.c_int, [P])]:
            fn = getattr(lib, f"plbm_gpu_{name}")
            fn.restype = res
            fn.argtypes = args
        lib.plbm_gpu_set_capture.argtypes = [C.c_void_p, C.c_int]
        lib.plbm_gpu_set_profiling.argtypes = [C.c_void_p, C.c_int]
        lib.plbm_gpu_kernel_stats.argtypes = [C.c_void_p, C.POINTER(KernelStats)]
        lib.plbm_gpu_reset_kernel_stats.argtypes = [C.c_void_p]
        lib.plbm_gpu_stream.argtypes = [C.c_void_p]
        lib.plbm_gpu_stream.restype = C.c_void_p
        lib.plbm_gpu_set_kernel_variant.argtypes = [C.c_void_p, C.c_int]
        if capture:
            self.set_capture(True)

    def set_capture(self, on: bool) -> None:
        if self.lib.plbm_gpu_set_capture(self._h, int(on)) != 0:
            raise RuntimeError("set_capture failed")

    def set_profiling(self, on: bool) -> None:
        self.lib.plbm_gpu_set_profiling(self._h, int(on))

    def kernel_stats(self) -> dict:
        k = KernelStats()
        self.lib.plbm_gpu_kernel_stats(self._h, C.byref(k))
        return {n: getattr(k, n) for n, _ in k._fields_}

    def reset_kernel_stats(self) -> None:
        self.lib.plbm_gpu_reset_kernel_stats(self._h)

    # ---- multi-rank protocol (include/plbm_gpu.h "multi-GPU") ----------------
    def prepare(self) -> None:
        if self.lib.plbm_gpu_prepare(self._h) != 0:
            raise RuntimeError("plbm_gpu_prepare failed (peers attached?)")

    def step_begin(self) -> None:
        err = Error()
        if self.lib.plbm_gpu_step_begin(self._h, C.byref(err)) != 0:
            raise EngineError(err)

    def step_main(self) -> None:
        err = Error()
        if self.lib.plbm_gpu_step_main(self._h, C.byref(err)) != 0:
            raise EngineError(err)

    def step_face(self) -> None:
        self.lib.plbm_gpu_step_face(self._h)

    def step_end(self, merged: "np.ndarray | None" = None) -> None:
        err = Error()
        ptr = None if merged is None else merged.ctypes.data_as(C.c_void_p)
        if self.lib.plbm_gpu_step_end(self._h, ptr, C.byref(err)) != 0:
            raise EngineError(err)

    def trigger_bytes(self) -> int:
        return self.lib.plbm_gpu_trigger_bytes(self._h)

    def triggers_device(self) -> int:
        return self.lib.plbm_gpu_triggers_device(self._h)

    def local_triggers(self) -> np.ndarray:
        out = np.zeros(self.trigger_bytes(), np.uint8)
        self.lib.plbm_gpu_local_triggers(self._h, out.ctypes.data_as(C.c_void_p), out.size)
        return out

    def ipc_handles(self) -> bytes:
        buf = (C.c_char * 256)()
        n = self.lib.plbm_gpu_ipc_handles(self._h, buf)
        if n <= 0:
            raise RuntimeError("plbm_gpu_ipc_handles failed")
        return bytes(buf[:n])

    def open_peer(self, rank: int, handles: bytes) -> None:
        buf = (C.c_char * len(handles)).from_buffer_copy(handles)
        if self.lib.plbm_gpu_open_peer(self._h, rank, buf) != 0:
            raise RuntimeError(f"plbm_gpu_open_peer({rank}) failed")

    def pool_pointers(self):
        """(population pool, psi-face pool, sync block) device pointers."""
        f, pf = C.c_void_p(), C.c_void_p()
        self.lib.plbm_gpu_pool_pointers(self._h, C.byref(f), C.byref(pf))
        return f.value, pf.value, self.lib.plbm_gpu_sync_block(self._h)

    def set_peer_pools(self, rank: int, pools) -> None:
        """Attach a same-process peer engine's pools (pool_pointers())."""
        if self.lib.plbm_gpu_set_peer_pools(self._h, rank, pools[0], pools[1]) != 0:
            raise RuntimeError("plbm_gpu_set_peer_pools failed")
        if len(pools) > 2 and self.lib.plbm_gpu_set_peer_sync(self._h, rank, pools[2]) != 0:
            raise RuntimeError("plbm_gpu_set_peer_sync failed")

    def tile_rank(self, coords) -> int:
        return self.lib.plbm_gpu_tile_rank(self._h, (C.c_int32 * 3)(*coords))

    def sync(self) -> None:
        self.lib.plbm_gpu_sync(self._h)

    def exchange_bytes(self) -> dict:
        """Bytes this rank reads from peer pools per step (NVLink), from the
        routing tables (plbm_gpu_exchange_bytes)."""
        out = (C.c_uint64 * 3)()
        self.lib.plbm_gpu_exchange_bytes.argtypes = [C.c_void_p, C.c_void_p]
        self.lib.plbm_gpu_exchange_bytes(self._h, out)
        return {"bytes_per_step": out[0], "remote_face_routes": out[1], "remote_edge_routes": out[2]}

    def gather_field(self, field: str, comp: int) -> np.ndarray:
        """iobench::gather_field (proj/src/dump.cpp:21-57): the domain grid,
        indexed [z, y, x]."""
        d = self.scenario.domain
        out = np.empty(d[0] * d[1] * d[2], np.float64)
        fn = self.lib.plbm_gpu_gather_field
        fn.restype = C.c_int
        fn.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_void_p]
        rc = fn(self._h, field.encode(), comp, out.ctypes.data_as(C.c_void_p))
        if rc != 0:
            raise RuntimeError(f"plbm_gpu_gather_field({field}, {comp}) failed: rc={rc}")
        return out.reshape(d[2], d[1], d[0])

    def set_kernel_variant(self, variant: int) -> None:
        """Fused-kernel variant (include/plbm_gpu.h): 0 = default, 1 = plain
        kernel, 21 / 22 = k_main_pc A/B variants, +100 / +200 modifiers."""
        if self.lib.plbm_gpu_set_kernel_variant(self._h, int(variant)) != 0:
            raise ValueError(f"unknown kernel variant {variant}")

    def stream(self) -> int:
        return self.lib.plbm_gpu_stream(self._h)

    def memory(self) -> dict:
        """Population pool footprint (plbm_gpu_memory): the address range and
        the bytes physically backed."""
        out = (C.c_uint64 * 5)()
        self.lib.plbm_gpu_memory.argtypes = [C.c_void_p, C.c_void_p]
        self.lib.plbm_gpu_memory(self._h, out)
        return {"pool_reserved_bytes": out[0], "pool_mapped_bytes": out[1], "granule_bytes": out[2],
                "map_host_ms": out[3] / 1e3, "map_wait_ms": out[4] / 1e3}


def gpu_engine(sc: Scenario, device: int = 0, capture: bool = False, rank: int = 0,
               world: int = 1, storage: str = "ab") -> GpuEngine:
    """storage "ab" (two population buffers) or "aa" (one buffer, A-A in place)."""
    return GpuEngine(sc, device, capture, rank, world, storage)
