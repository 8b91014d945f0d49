"""hetplan_b200 (the reference CLI on the engine) against the reference's own
cmd_plan / cmd_estimate / cmd_compare / cmd_scenario (cli.cpp:76-283) run by
oracle/_ref/ref_dump on the same command lines (tests/golden/cli/cases.json):
exit codes, stdout, stderr and every written file byte for byte, except the
wall-clock field of the plan report. Scenario cases need no GPU."""
import json
import os
import re
import subprocess
import tempfile

import pytest

from golden_util import load

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2512_12476_b200", "hetplan_b200")
GPU_FREE = ("scenario",)


def _norm(text: str) -> str:
    text = re.sub(r'"wall_clock_s": [^,\n]+', '"wall_clock_s": 0', text)
    return re.sub(r"(?m)^wall clock .*\n", "", text)


def _scratch():
    """a scratch dir named like ref_dump's mkdtemp("/tmp/hpg_cli_XXXXXX"): the
    text reports pad paths to fixed widths, so the length must match"""
    import random
    import string
    while True:
        d = "/tmp/hpg_cli_" + "".join(random.choices(string.ascii_letters + string.digits, k=6))
        try:
            os.mkdir(d)
            return d
        except FileExistsError:
            continue


def _run_cases(cases):
    import shutil
    bad = []
    tmp = _scratch()
    try:
        for c in cases:
            for fn, text in c.get("inputs", {}).items():  # defective input files
                with open(os.path.join(tmp, fn), "w") as f:
                    f.write(text)
            if c["name"] == "estimate_unknown_device":
                with open(os.path.join(tmp, "p1.json")) as f:
                    t = f.read()
                with open(os.path.join(tmp, "bad.json"), "w") as f:
                    f.write(t.replace('"a100-00"', '"zz-99"', 1))
            args = [a.replace("{tmp}", tmp) for a in c["args"]]
            r = subprocess.run([CLI] + args, cwd=ROOT, capture_output=True, text=True,
                               timeout=600)
            out, err = r.stdout.replace(tmp, "{tmp}"), r.stderr.replace(tmp, "{tmp}")
            if r.returncode != c["rc"]:
                bad.append(f"{c['name']}: rc {r.returncode} != {c['rc']} ({err.strip()})")
                continue
            if _norm(out) != _norm(c["stdout"]):
                bad.append(f"{c['name']}: stdout differs\n--- got\n{out}\n--- want\n{c['stdout']}")
            if err != c["stderr"]:
                bad.append(f"{c['name']}: stderr {err!r} != {c['stderr']!r}")
            for fn, want in c["files"].items():
                with open(os.path.join(tmp, fn)) as f:
                    got = f.read().replace(tmp, "{tmp}")
                if got != want:
                    bad.append(f"{c['name']}: file {fn} differs")
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    return bad


def _cases(gpu: bool):
    cases = load("cli/cases.json")["cases"]
    return [c for c in cases if (c["args"][0] in GPU_FREE) != gpu]


def test_cli_scenarios_identical():
    """scenario synthesis (topology.cpp:222-391) and its error paths"""
    if not os.path.exists(CLI):
        pytest.skip("hetplan_b200 not built")
    bad = _run_cases(_cases(gpu=False))
    assert not bad, "\n".join(bad)


def test_cli_fleet_reproduces_config4():
    """the fleet generator regenerates fixtures/c4.topology.json"""
    if not os.path.exists(CLI):
        pytest.skip("hetplan_b200 not built")
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "fleet.json")
        r = subprocess.run([CLI, "scenario", "--id", "fleet", "--seed", "7", "--out", out],
                           capture_output=True, text=True, timeout=60)
        assert r.returncode == 0, r.stderr
        with open(out) as f, open(os.path.join(ROOT, "fixtures", "c4.topology.json")) as g:
            assert f.read() == g.read()


@pytest.mark.gpu
def test_cli_plan_estimate_compare_identical():
    """plan (json/text, knobs file, budget/seed flags), estimate, compare and
    their error paths (defective plans, topologies and workflows: resolve_plan,
    DeviceTopology::make and build_workflow validation, JSON schema errors):
    byte-identical to the reference CLI"""
    bad = _run_cases(load("cli/cases.json")["cases"])
    assert not bad, "\n".join(bad[:10])
