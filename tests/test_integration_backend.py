"""The drop-in proven at link level: the reference's own
collect() (simoracle.cpp:143-161, compiled from /root/reference by
oracle/build_ref.sh) sweeps the B200 executor through the reference-side
binding integration/b200_backend.cpp, which replaces the simulator's run /
kernel_max_wgsize / is_refused.  The binary checks the reference's collect
contract (tests/test_simoracle.cpp:183-250) on real measurements."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "b200_collect"


@pytest.mark.gpu
def test_reference_collect_through_b200_backend():
    if not BIN.exists():
        pytest.skip("oracle/_ref/b200_collect not built (needs /root/reference at build time)")
    proc = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0 and proc.stdout.strip().endswith("OK"), proc.stdout + proc.stderr


def test_binding_resolves_the_simulator_symbols():
    """The linked binary carries exactly one definition of each replaced
    function (the binding's), the simulator's being weak."""
    if not BIN.exists():
        pytest.skip("oracle/_ref/b200_collect not built")
    out = subprocess.run(["nm", "-C", str(BIN)], capture_output=True, text=True).stdout
    for fn in ("wgtune::run(", "wgtune::is_refused(", "wgtune::kernel_max_wgsize("):
        defs = [ln for ln in out.splitlines() if fn in ln and " T " in ln]
        assert len(defs) == 1, (fn, defs)
