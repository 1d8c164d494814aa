"""The C++ drop-in shim (include/ibm_b200.hpp): compiles against the C ABI on the CPU; on the GPU
the example driver runs the reference's call sequence end to end."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "drop_in")


def _build():
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "drop_in.cpp"), "-L" + os.path.join(ROOT, "paper_1109_3524_b200"),
           "-libmgpu", "-Wl,-rpath," + os.path.join(ROOT, "paper_1109_3524_b200"), "-o", EXE]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_cpp_shim_compiles_and_links():
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_cpp_shim_runs_reference_sequence():
    _build()
    r = subprocess.run([EXE, os.path.join(ROOT, "cases", "cylinder_re40_smoke.cfg")], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "converged" in r.stdout and "invalid_argument" in r.stdout
    assert r.stdout.count("ok=1") == 3
    assert "checkpoint resume bitwise identical" in r.stdout


ACC = os.path.join(ROOT, "build", "acceptance_b200")


def _build_acceptance():
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(ROOT, "tests", "cpp"), os.path.join(ROOT, "tests", "cpp", "acceptance_b200.cpp"),
           "-L" + os.path.join(ROOT, "paper_1109_3524_b200"), "-libmgpu",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_1109_3524_b200"), "-o", ACC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_acceptance_driver_compiles():
    """The reference acceptance criteria 5/7/8/9 (acceptance.cpp:216-410) written against the shim's
    reference-named API compile with only the include and namespace switched."""
    _build_acceptance()


@pytest.mark.gpu
def test_acceptance_criteria_pass_through_shim():
    _build_acceptance()
    r = subprocess.run([ACC, os.path.join(ROOT, "cases")], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    for crit in ("5", "7", "8", "9", "x"):
        assert f"PASS criterion {crit}:" in r.stdout
