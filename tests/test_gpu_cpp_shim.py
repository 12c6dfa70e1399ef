"""GPU: the C++ drop-in shim (include/memplan_b200.hpp) against the reference
library, both driven through the reference's own memplan::Graph
(tests/cpp/shim_parity.cpp; built by __graft_entry__.build())."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "_bin", "shim_parity")


def test_cpp_shim_matches_reference(golden, built, tmp_path):
    if not os.path.exists(BIN):
        pytest.fail("tests/cpp/_bin/shim_parity missing: build() on a host with /root/reference")
    files = []
    for rec in golden["graphs"]:
        p = tmp_path / (rec["name"] + ".json")
        p.write_text(rec["graph_json"])
        files.append(str(p))
    out = subprocess.run([BIN, *files], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("OK "), out.stdout
    assert int(out.stdout.split()[1]) > 1000
