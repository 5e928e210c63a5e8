"""Build recipe for the product library (libplbm_gpu.so) and the parity checkers.

    python -m paper_1510_03560_b200.build            # product + oracle (+ reference shim)

The product is compiled for sm_100a only.  -fmad=false keeps every FP64
multiply and add separately rounded (the reference's x86-64 -O3 build has no
FMA), which is what makes the device results bit-identical to the reference.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(REPO, "include")
LIB = os.path.join(HERE, "libplbm_gpu.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "--expt-relaxed-constexpr",
    "-shared",
]


def _sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))]


def needs_rebuild() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = _sources() + [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)]
    return any(os.path.getmtime(p) > t for p in deps)


def build_gpu(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_rebuild():
        return LIB
    cmd = ["nvcc", *NVCC_FLAGS, "-I", INCLUDE, "-I", CSRC,
           os.path.join(CSRC, "engine.cu"), "-o", LIB + ".tmp", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed for libplbm_gpu.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    with open(os.path.join(HERE, "ptxas_report.txt"), "w") as fh:
        fh.write(r.stderr)
    return LIB


def build_exp(out: str, defines) -> str:
    """Measurement / A-B builds (not the product): engine.cu with extra -D
    flags into `out`, loaded through PLBM_GPU_LIB.  E.g.
        python -m paper_1510_03560_b200.build --exp build/exp/libphases.so PLBM_PHASES PLBM_ONLY_E32C2"""
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    cmd = ["nvcc", *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-I", CSRC,
           os.path.join(CSRC, "engine.cu"), "-o", out, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed for {out}")
    with open(out + ".ptxas.txt", "w") as fh:
        fh.write(r.stderr)
    return out


def build_oracle() -> None:
    """Parity checkers (test infrastructure): the C restatement always, the
    reference itself only where /root/reference exists (this container)."""
    odir = os.path.join(REPO, "oracle")
    subprocess.run(["make", "-s", "-C", odir, "oracle"], check=True)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", odir, "ref"], check=True)


def build_integration() -> None:
    """The reference's driver linked against libplbm_gpu.so
    (integration/plbm_gpu_run.cpp), where /root/reference exists."""
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "integration")], check=True)


if __name__ == "__main__":
    if "--exp" in sys.argv:
        i = sys.argv.index("--exp")
        print(build_exp(sys.argv[i + 1], sys.argv[i + 2:]))
        sys.exit(0)
    build_gpu(force="--force" in sys.argv, verbose=True)
    build_oracle()
    build_integration()
    print(LIB)
