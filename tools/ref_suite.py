"""Run the reference's own unit tests against this package (drop-in check).

`hybridsea` (and its submodules) are aliased to `paper_2511_02852_b200.host`
(the numpy face; the package's own modules where results are host values), then
pytest runs the reference test modules for the hot path from a staged copy
of the reference test suite (baseline/_ref/tests: git-ignored, staged from
/root/reference/pkg/tests by `python tools/ref_suite.py --stage` where the
reference exists; it travels to the GPU box like baseline/_ref).  Writes a
per-test outcome table (json) with the first line of every failure.

    python tools/ref_suite.py [--out gpurun_out/ref_suite.json] [modules...]
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
TESTS = os.path.join(ROOT, "baseline", "_ref", "tests")
HOT = ["test_spectrum", "test_fft_background", "test_particles", "test_patch_synthesis", "test_coupling",
       "test_harness", "test_config"]
# hybridsea.<m> -> the host face (numpy results) where it has one, else the package module
SUBMODULES = {"config": "config", "coupling": "host.coupling", "errors": "errors",
              "fft_background": "host.fft_background", "harness": "host.harness", "interaction": "interaction",
              "particles": "particles", "patch_synthesis": "host.patch_synthesis", "spectrum": "spectrum"}


def alias() -> None:
    import importlib
    pkg = importlib.import_module("paper_2511_02852_b200.host")
    sys.modules["hybridsea"] = pkg
    for m, target in SUBMODULES.items():
        sys.modules[f"hybridsea.{m}"] = importlib.import_module(f"paper_2511_02852_b200.{target}")


class Collect:
    def __init__(self):
        self.rows = {}

    def pytest_runtest_logreport(self, report):
        if report.when == "call" or (report.when == "setup" and report.outcome != "passed"):
            msg = ""
            if report.outcome == "failed":
                text = str(report.longrepr)
                lines = [ln for ln in text.splitlines() if ln.startswith("E ")]
                msg = (lines[0] if lines else text.splitlines()[-1])[:300]
            self.rows[report.nodeid] = {"outcome": report.outcome, "error": msg}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--stage", action="store_true", help="copy /root/reference/pkg/tests to baseline/_ref/tests")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "ref_suite.json"))
    ap.add_argument("modules", nargs="*", default=HOT)
    args = ap.parse_args()
    if args.stage:
        os.makedirs(TESTS, exist_ok=True)
        src = "/root/reference/pkg/tests"
        for f in os.listdir(src):
            if f.endswith(".py"):
                shutil.copy(os.path.join(src, f), TESTS)
        print("staged", TESTS)
        return 0
    if not os.path.isdir(TESTS):
        print(json.dumps({"unavailable": "reference tests not staged in baseline/_ref/tests"}))
        return 0
    alias()
    import pytest
    sys.path.insert(0, TESTS)
    col = Collect()
    files = [os.path.join(TESTS, m + ".py") for m in args.modules]
    rc = pytest.main(["-q", "-p", "no:cacheprovider", "-p", "no:randomly", "--rootdir", TESTS, *files],
                     plugins=[col])
    summary = {}
    for nid, r in col.rows.items():
        summary.setdefault(r["outcome"], 0)
        summary[r["outcome"]] += 1
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"summary": summary, "tests": col.rows}, open(args.out, "w"), indent=1)
    print(json.dumps(summary))
    return 0 if rc in (0, 1) else int(rc)


if __name__ == "__main__":
    sys.exit(main())
