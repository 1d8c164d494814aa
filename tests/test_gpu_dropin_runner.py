"""The drop-in proof at the reference's own top level: oracle/_ref/run_case_b200 is the reference's
parse_config + run_case (runner.hpp:77-164) compiled from its headers with ONE patched line — the
Stepper in run_case declared as ibm_b200::Stepper. The reference's run loop, force
writer, vorticity snapshots and checkpoints drive the B200 path; forces.csv must follow the
reference Stepper's per-step forces (1e-6) and the final checkpoint must be readable by the
reference (io.hpp:112-145)."""
import os
import subprocess

import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "run_case_b200")


@pytest.mark.parametrize("name,steps", [("cylinder_re40_smoke", 6), ("flapping_smoke", 6)])
def test_reference_run_case_on_the_device_stepper(ref, tmp_path, name, steps):
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/run_case_b200 not built (needs /root/reference at build time)")
    out = tmp_path / "out"
    r = subprocess.run([EXE, H.case(name), str(out), str(steps)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert f"steps {steps}" in r.stdout
    rows = (out / "forces.csv").read_text().splitlines()
    assert len(rows) == steps + 1
    rc = ref.case(H.case(name))
    for row in rows[1:]:
        rc.step()
        t, fx, fy, cd, cl = map(float, row.split(","))
        fr = rc.forces()
        assert abs(t - rc.time()) <= 1e-12
        assert abs(cd - fr["cd"]) <= 1e-6 * max(abs(fr["cd"]), 1e-3), (t, cd, fr["cd"])
        assert abs(cl - fr["cl"]) <= 1e-6 * max(abs(fr["cd"]), 1e-3), (t, cl, fr["cl"])
    # the reference resumes from the device run's final checkpoint and stays in step
    rc2 = ref.case(H.case(name))
    rc2.read_checkpoint(str(out / "checkpoint_final.txt"))
    assert abs(rc2.time() - rc.time()) <= 1e-12
    assert H.rel_err(rc2.state("q"), rc.state("q")) <= 1e-6
    assert (out / "vorticity_final.txt").read_text().startswith("# vorticity")
