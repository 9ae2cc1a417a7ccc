"""Drop-in conformance: the reference's own hot-path tests run against the B200 backend.

SURVEY §4 ("Reusing the reference suite as the drop-in's conformance suite"):
the unmodified reference test files (baseline/_ref/walkvec_tests, installed by
baseline/install_ref.sh) run in a subprocess with tests/conformance_plugin.py,
which calls ``install()`` before collection, so every ``random_walks``,
``bfs_walks``, ``train``, ``load_data`` and writer call in those tests goes to
the device implementations.  Two modes:

* ``fp64:numpy`` -- fp64 store replaying the reference's own numpy streams:
  the reference's results to fp64 rounding, so every hot-path test must pass
  except the known deviations below;
* ``fp64:device`` -- the default drop-in (fp64 store, device Feistel/Philox
  streams): tests that pin the reference's exact numpy streams may differ.

Expected deviations (each with its reason) are listed in EXPECTED; any other
failure fails this test (an expected one may pass: it is timing-dependent).
The call counters prove the backend ran.
"""

import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF_TESTS = ROOT / "baseline" / "_ref" / "walkvec_tests"
FILES = ["test_walks.py", "test_w2v.py", "test_pipeline.py", "test_acceptance.py"]

# node id -> reason; per mode
SCALING = ("CPU-shaped timing ratios (SURVEY §4 item 6): train time(10 epochs)/time(5 epochs) in [1.5, 2.5] on a "
           "~8k-pair corpus -- on the GPU both runs take milliseconds and the per-call setup (parameter store, "
           "workspace, CUDA-graph capture) is a fixed cost, so the ratio falls below 1.5; the walk-time ratio "
           "(1000 vs 100 walks per root) in the same test is within its band")
EXPECTED = {
    "fp64:numpy": {"test_acceptance.py::test_scaling_properties": SCALING},
    "fp64:device": {"test_acceptance.py::test_scaling_properties": SCALING},
}
BACKEND_CALLS = ("random_walks", "bfs_walks", "train")  # swapped attributes (package, walks, w2v, pipeline)


def _run(mode, tmp_path):
    xml = tmp_path / "junit.xml"
    calls = tmp_path / "calls.json"
    env = dict(os.environ, WV_CONFORMANCE=mode, WV_CONFORMANCE_CALLS=str(calls), PYTHONDONTWRITEBYTECODE="1",
               PYTHONPATH=os.pathsep.join([str(ROOT / "tests"), str(ROOT), str(ROOT / "baseline" / "_ref")]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "conformance_plugin", "-p", "no:cacheprovider",
           f"--junitxml={xml}", "--rootdir", str(REF_TESTS), *[str(REF_TESTS / f) for f in FILES]]
    proc = subprocess.run(cmd, cwd=str(REF_TESTS), env=env, capture_output=True, text=True, timeout=3000)
    assert xml.exists(), proc.stdout[-3000:] + proc.stderr[-3000:]
    outcomes = {}
    for case in ET.parse(xml).getroot().iter("testcase"):
        cls = case.get("classname", "")
        mod = cls.split(".")[0] + ".py"
        rest = ".".join(cls.split(".")[1:])
        node = f"{mod}::{rest + '::' if rest else ''}{case.get('name')}"
        kind = "passed"
        for child in case:
            if child.tag in ("failure", "error"):
                kind = "failed"
            elif child.tag == "skipped":
                kind = "skipped"
        outcomes[node] = kind
    return outcomes, json.loads(calls.read_text()) if calls.exists() else {}, proc


@pytest.mark.skipif(not (REF_TESTS / "conftest.py").exists(),
                    reason="baseline/_ref not installed (run baseline/install_ref.sh)")
@pytest.mark.parametrize("mode", ["fp64:numpy", "fp64:device"])
def test_reference_suite_through_install(mode, tmp_path):
    outcomes, calls, proc = _run(mode, tmp_path)
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    report = {"mode": mode, "outcomes": outcomes, "calls": calls,
              "summary": {k: sum(v == k for v in outcomes.values()) for k in ("passed", "failed", "skipped")}}
    (ROOT / "gpurun_out" / f"conformance_{mode.replace(':', '_')}.json").write_text(json.dumps(report, indent=1))
    failed = {n for n, k in outcomes.items() if k == "failed"}
    expected = EXPECTED[mode]

    def matches(node):
        return any(node == e or node.startswith(e + "[") or node.endswith("::" + e.split("::")[-1]) and
                   node.split("::")[0] == e.split("::")[0] for e in expected)

    unexpected = sorted(n for n in failed if not matches(n))
    assert not unexpected, (unexpected, proc.stdout[-4000:])
    assert report["summary"]["passed"] >= 100, report["summary"]
    for name in BACKEND_CALLS:
        assert sum(v for k, v in calls.items() if k.endswith("." + name)) > 0, (name, calls)
