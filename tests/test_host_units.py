"""CPU tests of host-side building blocks (no GPU): the exact fast remainder
used by the candidate generator, the Rng stream pinned to the reference and
its jump-ahead."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def host_units(tmp_path_factory):
    exe = tmp_path_factory.mktemp("hu") / "host_units"
    subprocess.run(["g++", "-std=c++20", "-O2", "-o", str(exe),
                    os.path.join(ROOT, "tests", "host_units.cpp")], check=True)
    return str(exe)


def test_fastmod_exact(host_units):
    out = subprocess.run([host_units, "42"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert "mismatches 0" in out.stdout


def test_rng_jump_ahead_exact(host_units):
    """x^D mod p (Berlekamp-Massey characteristic polynomial) applied to a
    state equals D draws: the device GA's init chunks start every lane there"""
    out = subprocess.run([host_units, "42"], capture_output=True, text=True)
    assert "jump mismatches 0" in out.stdout, out.stdout


def test_rng_stream_matches_reference(host_units):
    with open(os.path.join(ROOT, "tests", "golden", "rng_pin.json")) as f:
        gold = json.load(f)
    for seed, want in gold.items():
        out = subprocess.run([host_units, seed], capture_output=True, text=True).stdout
        lines = [ln for ln in out.splitlines() if ln.startswith(("draws", "fork7"))]
        assert lines == want, (seed, lines, want)
