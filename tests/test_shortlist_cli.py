"""The model's shortlist (autotune.hpp shortlist_classify / shortlist_regress,
CLI `wgtb predict --shortlist N`) on the committed bundle, offline (device
descriptor from results/b200/device.json, no GPU): the first entry is the
plain Algorithm-1 prediction, entries are distinct legal sizes, a longer
list extends a shorter one, and the forest's vote ranking brings in the
labels the single prediction cannot (f32 and i32 grids share fv1 features)."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
B = ROOT / "results" / "b200"
WGTB = ROOT / "paper_1511_02490_b200" / "lib" / "wgtb"

pytestmark = pytest.mark.skipif(not WGTB.exists(), reason="wgtb CLI not built")


def predict(kernel: str, ds: str, n: int = 0, model: Path = B / "model.json"):
    cmd = [str(WGTB), "predict", "--model", str(model), "--device", f"json:{B / 'device.json'}",
           "--kernel-json", str(B / "descriptors" / "kernels" / f"{kernel}.json"), "--dataset", ds]
    if n:
        cmd += ["--shortlist", str(n)]
    v = list(map(int, subprocess.run(cmd, capture_output=True, text=True, check=True).stdout.split()))
    return list(zip(v[0::2], v[1::2]))


@pytest.mark.parametrize("kernel,ds", [("he", "16384x16384-FLOAT32-FLOAT32"), ("gol", "8192x8192-INT32-INT32"),
                                       ("boxmean-5130", "4096x4096-FLOAT32-FLOAT32")])
def test_shortlist_extends_the_prediction(kernel, ds):
    one = predict(kernel, ds)
    sl8 = predict(kernel, ds, 8)
    sl3 = predict(kernel, ds, 3)
    assert len(one) == 1 and sl8[0] == one[0]
    assert sl3 == sl8[:3]
    assert len(sl8) == 8 and len(set(sl8)) == 8
    for wc, wr in sl8:
        assert 2 <= wc and 2 <= wr and wc * wr <= 1024 and wc % 2 == 0 and wr % 2 == 0


def test_shortlist_holds_both_labels_of_an_fv1_collision():
    # he 16384^2: the f32 scenario's oracle (232x4 in the 30-observation
    # re-sweep) and the i32 scenario's (48x8) share one fv1 feature vector;
    # the single prediction answers the i32 label for both
    f32 = predict("he", "16384x16384-FLOAT32-FLOAT32", 8)
    i32 = predict("he", "16384x16384-INT32-INT32", 8)
    assert f32 == i32
    assert (48, 8) in f32 and (232, 4) in f32


def test_shortlist_rejects_nonpositive_n():
    with pytest.raises(subprocess.CalledProcessError):
        predict("he", "1024x1024-FLOAT32-FLOAT32", -1)
