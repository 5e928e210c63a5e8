"""Compare an engine's state with tests/golden/golden_states.json (produced by
the reference itself, see tests/golden/make_golden.py)."""
import json
import os

from tests.golden.make_golden import state_digest

HERE = os.path.dirname(os.path.abspath(__file__))


def load_golden():
    with open(os.path.join(HERE, "golden", "golden_states.json")) as fh:
        return json.load(fh)


def assert_matches_golden(eng, name):
    g = load_golden()[name]
    d = state_digest(eng)
    d = json.loads(json.dumps(d))  # normalise tuples -> lists
    assert d["counters"] == g["counters"], (d["counters"], g["counters"])
    assert d["creation_log"] == g["creation_log"]
    assert d["tiles"] == g["tiles"]
    bad = [k for k in g["fields"] if d["fields"].get(k) != g["fields"][k]]
    assert not bad, f"{len(bad)} fields differ from the reference golden state, e.g. {bad[:5]}"
