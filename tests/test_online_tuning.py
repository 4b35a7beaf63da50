"""Online tuning: wgtb_launch_tuned / Stencil<T>::
autotuned - the trained model proposes the workgroup size per session, the
launch runs it, and refused sizes are fed back so the model re-proposes
(reference serve.cpp:123-164: a session's refused set grows, the proposal
never repeats a refused size)."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1511_02490_b200 import Stencil  # noqa: E402
from paper_1511_02490_b200 import autotune  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
MODEL = ROOT / "results" / "b200" / "model.json"
KERNELS = ROOT / "results" / "b200" / "descriptors" / "kernels"


@pytest.fixture(autouse=True)
def fresh_sessions():
    autotune.Tuned.reset()
    yield
    autotune.Tuned.reset()


def test_first_proposal_is_the_prediction_and_output_is_exact():
    st = Stencil(op="heat", dtype="float32", border="nearest")
    x = np.random.default_rng(3).random((1024, 1024)).astype(np.float32)
    a = torch.from_numpy(x).cuda()
    b = torch.empty_like(a)
    tuned = autotune.Tuned(st, KERNELS / "he.json", MODEL)
    wc, wr = tuned(a, b)
    torch.cuda.synchronize()
    pred = autotune.predict(st, 1024, 1024, KERNELS / "he.json", MODEL)
    assert (wc, wr) == (pred["wc"], pred["wr"])
    assert tuned.last[2] == 1
    assert b.cpu().numpy().tobytes() == O.stencil(O.desc_from_stencil(st), x).tobytes()
    # the session is cached: no new proposal for the same grid
    tuned(a, b)
    assert tuned.last == (wc, wr, 1)


def test_refusal_feedback_reproposes_and_never_repeats():
    st = Stencil(op="gol", dtype="int32")
    x = (np.random.default_rng(4).random((512, 768)) < 0.4).astype(np.int32)
    a = torch.from_numpy(x).cuda()
    b = torch.empty_like(a)
    want = O.stencil(O.desc_from_stencil(st), x)
    tuned = autotune.Tuned(st, KERNELS / "gol.json", MODEL)
    seen = []
    for i in range(6):
        wc, wr = tuned(a, b)
        torch.cuda.synchronize()
        assert b.cpu().numpy().tobytes() == want.tobytes()
        assert (wc, wr) not in seen, "a refused size was proposed again"
        assert tuned.last[2] == i + 1
        seen.append((wc, wr))
        tuned.refuse(768, 512, wc, wr)  # forced refusal of the size that ran
    # another grid is another session: back to one proposal
    a2 = torch.from_numpy(np.ascontiguousarray(x[:256])).cuda()
    b2 = torch.empty_like(a2)
    tuned(a2, b2)
    assert tuned.last[2] == 1


def test_shortlist_leads_with_the_prediction_and_is_legal():
    st = Stencil(op="heat", dtype="float32", border="nearest")
    pred = autotune.predict(st, 4096, 4096, KERNELS / "he.json", MODEL)
    sl = autotune.shortlist(st, 4096, 4096, KERNELS / "he.json", MODEL, n=8)
    assert len(sl) == 8 and len(set(sl)) == 8
    assert sl[0] == (pred["wc"], pred["wr"])
    for wc, wr in sl:
        assert wc * wr <= 1024 and wc % 2 == 0 and wr % 2 == 0
    # a one-size shortlist is the prediction alone
    assert autotune.shortlist(st, 4096, 4096, KERNELS / "he.json", MODEL, n=1) == sl[:1]


def test_tune_measured_picks_the_fastest_of_the_shortlist_and_is_exact():
    st = Stencil(op="heat", dtype="float32", border="nearest")
    x = np.random.default_rng(5).random((2048, 2048)).astype(np.float32)
    a = torch.from_numpy(x).cuda()
    b = torch.empty_like(a)
    sl = autotune.shortlist(st, 2048, 2048, KERNELS / "he.json", MODEL, n=6)
    r = autotune.tune_measured(st, a, b, KERNELS / "he.json", MODEL, n=6, samples=3)
    assert r["timed"] == len(sl) and (r["wc"], r["wr"]) in sl and r["best_ms"] > 0
    one = autotune.tune_measured(st, a, b, KERNELS / "he.json", MODEL, n=1, samples=3)
    assert (one["wc"], one["wr"]) == sl[0] and one["timed"] == 1
    # the chosen size runs the stencil exactly
    st(a, b, wc=r["wc"], wr=r["wr"])
    torch.cuda.synchronize()
    assert b.cpu().numpy().tobytes() == O.stencil(O.desc_from_stencil(st), x).tobytes()
    with pytest.raises(RuntimeError):
        autotune.tune_measured(st, a, b, KERNELS / "he.json", MODEL, n=0)
