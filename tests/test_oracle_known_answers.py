"""Known-answer rows the reference's own tests pin (test_engine.py:141-183, 224-248;
test_exprlang.py:149-161; test_acceptance.py:122-124), checked against the oracle."""
import math

import numpy as np

from oracle import parallel as OP, recurrent as OR
from paper_2502_15349_b200 import spec as S


def _spec(name, **kw):
    base = dict(heads=1, seq_q=1, seq_k=2, d_qk=1, d_v=2)
    base.update(kw)
    return S.builtin(name, **base)


def test_softmax_row_quarter_three_quarters():
    # scores [0, ln 3] -> probabilities [1/4, 3/4]  (test_engine.py:163-173)
    sp = _spec("softmax")
    q = np.ones((1, 1, 1, 1))
    k = np.array([0.0, math.log(3.0)]).reshape(1, 1, 2, 1)   # q_mod divides by sqrt(1) = 1
    v = np.eye(2).reshape(1, 1, 2, 2)
    for bk in (1, 2):
        o = OP.tiled_forward(sp, {"q": q, "k": k, "v": v}, 1, bk)
        assert np.allclose(o[0, 0, 0], [0.25, 0.75], atol=1e-15)


def test_fully_masked_row_is_zero():
    # strict mask kills row 0 entirely -> output 0, LSE -inf (test_engine.py:233-248)
    sp = S.builtin("softmax", heads=1, seq=4, d_qk=2, d_v=2)
    sp = S.AttentionSpec(sp.name, sp.pattern, sp.dims, q_mod=sp.q_mod, rownorm=sp.rownorm,
                         score_mods=(S.mod("where(kidx < qidx, s, -inf)", "s", ismask=True),))
    rng = np.random.default_rng(0)
    arrays = {n: rng.uniform(-1, 1, (1, 1, 4, 2)) for n in "qkv"}
    arrays["qidx"] = np.arange(4.0).reshape(1, 1, 4, 1)
    arrays["kidx"] = np.arange(4.0).reshape(1, 1, 1, 4)
    o = OP.tiled_forward(sp, arrays, 2, 2)
    assert np.all(o[0, 0, 0] == 0.0)
    assert OP.lse_rows(sp, arrays)[0, 0, 0] == -math.inf


def test_abssum_clamp_rows():
    # retention-parallel: row [0.5, -2] -> /2.5 ; row sum below 1 passes through
    # (test_engine.py:141-152, test_acceptance.py:122-124)
    sp = S.builtin("retention-parallel", heads=1, seq_q=1, seq_k=2, d_qk=1, d_v=2, gamma=1.0)
    arrays = {"q": np.ones((1, 1, 1, 1)), "k": np.array([0.5, -2.0]).reshape(1, 1, 2, 1),
              "v": np.eye(2).reshape(1, 1, 2, 2),
              "mask": np.ones((1, 1, 1, 2))}
    o = OP.tiled_forward(sp, arrays, 1, 1)
    assert np.allclose(o[0, 0, 0], [0.2, -0.8], atol=1e-15)
    arrays["k"] = np.array([0.3, 0.2]).reshape(1, 1, 2, 1)
    o = OP.tiled_forward(sp, arrays, 1, 1)
    assert np.allclose(o[0, 0, 0], [0.3, 0.2], atol=1e-15)


def test_first_recurrent_step_is_outer_product():
    # o_0 = q_0 (k_0^T v_0)  (test_engine.py:176-183)
    sp = S.builtin("retention-recurrent", heads=1, seq=3, d_qk=2, d_v=3)
    rng = np.random.default_rng(1)
    arrays = {"q": rng.uniform(-1, 1, (1, 1, 3, 2)), "k": rng.uniform(-1, 1, (1, 1, 3, 2)),
              "v": rng.uniform(-1, 1, (1, 1, 3, 3)), "decay": np.full((1, 1, 3, 1), 0.9)}
    o = OR.step_forward(sp, arrays)
    q0 = arrays["q"][0, 0, 0] / math.sqrt(2)
    want = q0 @ np.outer(arrays["k"][0, 0, 0], arrays["v"][0, 0, 0])
    assert np.allclose(o[0, 0, 0], want, atol=1e-15)
    assert np.allclose(OR.chunk_forward(sp, arrays, 2), o, atol=1e-14)


def test_decode_row_single_query():
    # seq_q = 1 decode row, unmasked (test_engine.py:224-230; top-left causal would
    # mask all but key 0 at decode)
    sp = S.builtin("softmax", heads=2, seq_q=1, seq_k=37, d_qk=8, d_v=8)
    rng = np.random.default_rng(2)
    arrays = {"q": rng.uniform(-1, 1, (1, 2, 1, 8)), "k": rng.uniform(-1, 1, (1, 2, 37, 8)),
              "v": rng.uniform(-1, 1, (1, 2, 37, 8))}
    assert np.allclose(OP.tiled_forward(sp, arrays, 1, 8), OP.naive_forward(sp, arrays),
                       atol=1e-14)
