"""bench.py sanity without a GPU: the driver runs it at round end on a fresh
box, so a Python-level error there costs the round's measurement.

* no function shadows a module-level function or import with a local name
  (an UnboundLocalError only shows on the GPU path otherwise);
* the reference arm runs end to end on the host (C1, a few steps)."""
import json
import os
import subprocess
import sys
import symtable

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(REPO, "bench.py")


def test_no_local_shadows_module_function():
    src = open(BENCH).read()
    top = symtable.symtable(src, BENCH, "exec")
    module_funcs = {s.get_name() for s in top.get_symbols()
                    if s.is_assigned() or s.is_imported()} | {c.get_name() for c in top.get_children()}
    bad = []

    def walk(tab):
        for ch in tab.get_children():
            if ch.get_type() == "function":
                for sym in ch.get_symbols():
                    n = sym.get_name()
                    if sym.is_local() and not sym.is_parameter() and n in module_funcs and sym.is_assigned():
                        if any(n == c.get_name() for c in top.get_children()):
                            bad.append((ch.get_name(), n))
            walk(ch)
    walk(top)
    assert not bad, f"locals shadowing module-level functions: {bad}"


def test_reference_arm_runs_on_host():
    from tests.conftest import have_ref
    if not have_ref():
        pytest.skip("reference shim not built")
    r = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--config", "c1", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["e2e"]["value"] == line["value"]
