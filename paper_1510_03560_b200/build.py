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


# translation units: the host engine + one kernel-instantiation unit per tile
# extent (csrc/dispatch.cuh), compiled in parallel and linked into one .so
UNITS = ["engine.cu", "inst_e8.cu", "inst_e16.cu", "inst_e32.cu", "inst_e64.cu"]


def needs_rebuild() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = _sources() + [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)]
    return any(os.path.getmtime(p) > t for p in deps)


def _compile_link(out: str, defines=(), units=UNITS) -> str:
    """nvcc -c every unit (in parallel) into build/obj/<out name>/, then link
    the shared library; ptxas -v output of all units is returned."""
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    odir = os.path.join(REPO, "build", "obj", os.path.basename(out).replace(".", "_"))
    os.makedirs(odir, exist_ok=True)
    procs = []
    for u in units:
        obj = os.path.join(odir, u.replace(".cu", ".o"))
        cmd = ["nvcc", *flags, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-I", CSRC, "-c",
               os.path.join(CSRC, u), "-o", obj]
        procs.append((u, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    report, objs = [], []
    for u, obj, pr in procs:
        so, se = pr.communicate()
        report.append(f"==== {u}\n{se}")
        if pr.returncode != 0:
            sys.stderr.write(so + se)
            raise RuntimeError(f"nvcc failed for {u}")
        objs.append(obj)
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", out + ".tmp", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"link failed for {out}")
    os.replace(out + ".tmp", out)
    return "".join(report)


def build_gpu(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_rebuild():
        return LIB
    report = _compile_link(LIB)
    if verbose:
        sys.stderr.write(report)
    with open(os.path.join(HERE, "ptxas_report.txt"), "w") as fh:
        fh.write(report)
    return LIB


def build_exp(out: str, defines) -> str:
    """Measurement / A-B builds (not the product): the units with extra -D
    flags into `out`, loaded through PLBM_GPU_LIB.  PLBM_ONLY_E32C2 builds the
    engine and the E = 32 unit only.  E.g.
        python -m paper_1510_03560_b200.build --exp build/exp/libphases.so PLBM_PHASES PLBM_ONLY_E32C2"""
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    units = ["engine.cu", "inst_e32.cu"] if "PLBM_ONLY_E32C2" in defines else UNITS
    report = _compile_link(os.path.abspath(out), defines, units)
    with open(out + ".ptxas.txt", "w") as fh:
        fh.write(report)
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
