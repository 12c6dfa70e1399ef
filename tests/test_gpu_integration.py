"""GPU: the drop-in at the reference's own call sites.

integration/Makefile builds the reference's planning entry point plan_graph
(proj/src/pipeline.cpp:296-324) twice: the unmodified reference
(integration/_bin/plan_graph_ref) and the reference with
integration/pipeline_b200.patch applied (plan_graph_b200), whose call sites -
the program-order baseline peak (pipeline.cpp:297-302), realized_lifetimes,
timeline_from_lifetimes, preallocate_pyramid, greedy_pack and
addresses_feasible - go through include/memplan_b200.hpp on the B200. Both
print the PlanResult (peak, savings, control edges, timed_out), the saved plan
and validate_plan's verdict; they must agree byte for byte. Graphs: the
reference fixtures and generated graphs from tests/golden/golden.json
(written to a temporary directory: /root/reference is not on the GPU box)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_bin")


def _run(exe, *args):
    r = subprocess.run([os.path.join(BIN, exe), *args], capture_output=True, text=True,
                       timeout=600)
    return r.returncode, r.stdout, r.stderr


def _untimed(out):
    """The saved plan's provenance carries wall-clock phase times (plan.cpp's
    schedule_seconds / placement_seconds): the only fields allowed to differ."""
    rc, text, err = out
    keep = [ln for ln in text.splitlines() if "_seconds" not in ln]
    return rc, "\n".join(keep), err


@pytest.fixture(scope="module")
def graph_files(golden, tmp_path_factory):
    if not os.path.exists(os.path.join(BIN, "plan_graph_b200")):
        pytest.skip("integration binaries not built (make -C integration)")
    d = tmp_path_factory.mktemp("graphs")
    out = []
    for rec in golden["graphs"]:
        p = d / (rec["name"] + ".json")
        p.write_text(rec["graph_json"])
        out.append((rec["name"], str(p)))
    return out


def test_plan_graph_identical_through_the_patched_call_sites(graph_files):
    compared = 0
    for name, path in graph_files:
        ref = _untimed(_run("plan_graph_ref", "plan", path))
        got = _untimed(_run("plan_graph_b200", "plan", path))
        # graphs past the internal solver limits need an external MILP solver, which
        # this image lacks: the reference and the patched build must then fail alike
        assert got == ref, name
        compared += ref[0] == 0
    assert compared >= 5          # the fixtures plan internally


def test_call_site_latency_program_order_peak(graph_files, tmp_path):
    """pipeline.cpp:297-302 for one order: the first B200 call includes upload and
    host analysis; cached calls are one launch + copies. Same peak as the reference."""
    import gzip
    import paper_2210_12924_b200 as mp
    cases = [(n, p) for n, p in graph_files if n in ("chain3", "training_mini")]
    for name in ("resnet50_b32", "bert_base_s512"):
        with gzip.open(os.path.join(ROOT, "workloads", "graphs", name + ".json.gz"), "rt") as f:
            p = tmp_path / (name + ".json")
            p.write_text(f.read())
        cases.append((name, str(p)))
    p = tmp_path / "training_like_L33333.json"
    p.write_text(mp.save_graph(mp.generate_graph("training_like", 33333, 8)))
    cases.append(("training_like_L33333", str(p)))
    rows = {}
    for name, path in cases:
        reps = "3" if name == "training_like_L33333" else "50"
        rc1, ref, _ = _run("plan_graph_ref", "peak", path, reps)
        rc2, got, _ = _run("plan_graph_b200", "peak", path, reps)
        assert rc1 == rc2 == 0, name
        r, g = json.loads(ref), json.loads(got)
        assert r["peak"] == g["peak"], name
        rows[name] = {"reference_us": r["cached_us"], "b200_first_us": g["first_us"],
                      "b200_cached_us": g["cached_us"]}
    print(json.dumps(rows))
