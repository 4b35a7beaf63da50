"""The strongest end-to-end oracle of SURVEY.md §8c: the reference's own
evaluate() (compiled from /root/reference into oracle/_ref/ref_evaluate),
fed the B200 re-sweep of the reference kernels (results/b200/real30: 30
observations per size, recorded contexts), must produce the same metric rows
as `wgtb evaluate` on the same files (time_ms, wall clock, excluded).  CPU
only; the heat and GoL scenarios (34) with 3 observations per size keep the
reference's run time (~90x ours on this data) to about a minute."""
from __future__ import annotations

import csv
import io
import lzma
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "oracle" / "_ref" / "ref_evaluate"
WGTB = ROOT / "paper_1511_02490_b200" / "lib" / "wgtb"
R30 = ROOT / "results" / "b200" / "real30"
DESC = ROOT / "results" / "b200" / "descriptors"


@pytest.fixture(scope="module")
def real30(tmp_path_factory):
    if not REF.exists():
        pytest.skip("oracle/_ref/ref_evaluate not built (needs /root/reference)")
    d = tmp_path_factory.mktemp("real30")
    desc = d / "desc"
    for sub in ("devices", "datasets"):
        shutil.copytree(DESC / sub, desc / sub)
    (desc / "kernels").mkdir()
    for k in ("he", "gol"):
        shutil.copy(DESC / "kernels" / f"{k}.json", desc / "kernels")
    for name in ("refused", "contexts"):
        (d / f"{name}.csv").write_bytes(lzma.decompress((R30 / f"{name}_real30.csv.xz").read_bytes()))
    # the first 3 of the 30 observations of every size: the same table for
    # both sides, 10x less text to parse per run
    seen = {}
    with lzma.open(R30 / "samples_real30.csv.xz", "rt") as f, open(d / "samples.csv", "w") as o:
        o.write(f.readline())
        for ln in f:
            key = ln.rsplit(",", 1)[0]
            n = seen.get(key, 0)
            if n < 3:
                o.write(ln)
            seen[key] = n + 1
    return d


def rows(text: str):
    out = []
    for r in csv.DictReader(io.StringIO(text)):
        r.pop("time_ms")
        out.append(r)
    return out


@pytest.mark.parametrize("technique", ["forest-nn", "nb-random", "speedup-reg"])
def test_reference_evaluate_equals_ours_on_b200_data(real30, tmp_path, technique):
    files = [str(real30 / f"{n}.csv") for n in ("samples", "refused", "contexts")]
    ref = subprocess.run([str(REF), str(real30 / "desc"), *files, technique, "kfold", "3", "0"], capture_output=True,
                         text=True, timeout=900)
    assert ref.returncode == 0, ref.stderr
    m = tmp_path / "m.csv"
    ours = subprocess.run([str(WGTB), "evaluate", "--scenarios", str(real30 / "desc"), "--samples", files[0],
                           "--refused", files[1], "--contexts", files[2], "--technique", technique,
                           "--partition", "kfold", "--folds", "3", "--seed", "0", "--metrics", str(m)],
                          capture_output=True, text=True, timeout=900)
    assert ours.returncode == 0, ours.stderr
    want, got = rows(ref.stdout), rows(m.read_text())
    assert len(want) == 34 and got == want
