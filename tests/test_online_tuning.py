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
