"""The C++ facade (include/semrank_b200.hpp) compiles against the C-ABI and
links the in-tree library, as a reference caller would."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2602_07309_b200", "lib")


def _build(tmp_path, name="facade_smoke"):
    exe = str(tmp_path / name)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", name + ".cpp"), "-L", LIBDIR,
                    "-lsemrank_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_facade_compiles_and_runs_host_api(tmp_path):
    out = subprocess.run([_build(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "facade ok" in out.stdout


@pytest.mark.gpu
def test_facade_scores_on_device(tmp_path):
    out = subprocess.run([_build(tmp_path), "gpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "relevance[0]=" in out.stdout


def test_acceptance_harness_compiles_against_facade(tmp_path):
    _build(tmp_path, "acceptance_facade")


@pytest.mark.gpu
def test_acceptance_criteria_1_and_4_through_facade(tmp_path):
    """acceptance_main.cpp:90-104 and 146-174 as the reference writes them,
    running on the device through the facade."""
    out = subprocess.run([_build(tmp_path, "acceptance_facade")], capture_output=True, text=True)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "criterion 1 PASS" in out.stdout and "criterion 4 PASS" in out.stdout
    assert "acceptance ok" in out.stdout
