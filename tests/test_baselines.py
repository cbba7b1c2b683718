"""Baseline sparsifiers (baselines.cpp:26-46).

CPU: the numpy restatement (oracle/oracle.py) against the reference's golden
vectors (tests/golden/baselines_golden.json, made by make_golden_baselines.py)
and, when oracle/_ref is built, against the unmodified reference on fresh
tie-heavy inputs. GPU: the device top-k / hard threshold through the C ABI,
bit-exact against both.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "baselines_golden.json")))
CASES = GOLD["cases"]


# ---------------------------------------------------------------- CPU -------
@pytest.mark.parametrize("case", CASES, ids=lambda c: c["tag"])
def test_numpy_restatement_matches_reference_golden(case):
    acc = np.array(case["acc"], np.float64)
    for t in case["topk"]:
        assert O.topk_select_np(acc, t["k"]).tolist() == t["idx"]
    for h in case["hard"]:
        assert O.hard_threshold_select_np(acc, h["delta"]).tolist() == h["idx"]


def test_numpy_restatement_rejects_k_out_of_range():
    # test_baselines.cpp:39-43
    with pytest.raises(ValueError, match="k out of range"):
        O.topk_select_np(np.array([1.0, 2.0]), 0)
    with pytest.raises(ValueError, match="k out of range"):
        O.topk_select_np(np.array([1.0, 2.0]), 3)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_numpy_restatement_matches_unmodified_reference_fresh_inputs():
    rng = np.random.default_rng(5)
    for trial in range(40):
        n = int(rng.integers(1, 3000))
        if trial % 2:
            acc = rng.choice([0.0, -0.0, 0.5, -0.5, 2.0], size=n)
        else:
            acc = rng.laplace(size=n)
        k = int(rng.integers(1, n + 1))
        assert np.array_equal(O.topk_select_np(acc, k), O.ref_topk_select(acc, k))
        d = float(rng.choice([0.0, 0.5, 1.0, 4.0]))
        assert np.array_equal(O.hard_threshold_select_np(acc, d),
                              O.ref_hard_threshold_select(acc, d))
    with pytest.raises(O.CheckError, match="k out of range"):
        O.ref_topk_select(np.array([1.0, 2.0]), 3)


def test_c_abi_argument_checks_without_gpu():
    # the range checks run before any CUDA call (engine.cu: baseline_select)
    import ctypes as C
    from paper_2402_13781_b200 import _abi as A
    from paper_2402_13781_b200._lib import lib
    L = lib()
    rc = L.exd_topk_select_device(None, 0, A.EXD_F32, 1, None, 1, None)
    assert rc == A.EXD_EINVAL and L.exd_last_error() == b"topk_select: k out of range"
    rc = L.exd_topk_select_device(None, 2, A.EXD_F32, 3, None, 3, None)
    assert rc == A.EXD_EINVAL and L.exd_last_error() == b"topk_select: k out of range"
    rc = L.exd_topk_select_device(None, 2, 7, 1, None, 1, None)
    assert rc == A.EXD_EINVAL and L.exd_last_error() == b"dtype out of range"
    cnt = C.c_int64(-1)
    rc = L.exd_hard_threshold_select_device(None, 0, A.EXD_F64, 0.5, None, 0, C.byref(cnt), None)
    assert rc == A.EXD_OK and cnt.value == 0


# ---------------------------------------------------------------- GPU -------
def _dev(acc, dtype):
    import torch
    return torch.tensor(np.asarray(acc, dtype=dtype), device="cuda:0")


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", CASES, ids=lambda c: c["tag"])
def test_device_matches_reference_golden(case, dtype):
    from paper_2402_13781_b200 import sparsim as S
    acc = np.array(case["acc"], np.float64)
    if dtype == np.float32 and not np.array_equal(acc.astype(np.float32).astype(np.float64), acc):
        pytest.skip("values not fp32-representable")
    a = _dev(acc, dtype)
    for t in case["topk"]:
        assert S.topk_select(a, t["k"]).cpu().numpy().tolist() == t["idx"], t["k"]
    for h in case["hard"]:
        assert S.hard_threshold_select(a, h["delta"]).cpu().numpy().tolist() == h["idx"], h["delta"]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n,k", [(11_200_000, 112_000), (6_200_000, 6_200), (1_000_003, 1),
                                 (1_000_003, 1_000_003), (4096 * 7 + 5, 9_000)])
def test_device_topk_vs_oracle_laplace(n, k, dtype):
    from paper_2402_13781_b200 import sparsim as S
    acc = np.random.default_rng(n + k).laplace(size=n).astype(dtype)
    got = S.topk_select(_dev(acc, dtype), k).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, O.topk_select_np(acc, k))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_device_topk_tie_heavy_crosses_tiles(dtype):
    # ties at the cut spread over many 4096-element tiles: the lower-index rule
    # must hold across tile and CTA boundaries
    from paper_2402_13781_b200 import sparsim as S
    rng = np.random.default_rng(11)
    n = 2_000_001
    acc = rng.choice(np.array([0.0, -0.0, 0.25, -0.25, 1.0, -1.0], dtype), size=n)
    for k in (1, 5, (acc != 0).sum() // 3 * 2, (acc != 0).sum() + 17, n):
        got = S.topk_select(_dev(acc, dtype), int(k)).cpu().numpy().astype(np.int64)
        assert np.array_equal(got, O.topk_select_np(acc, int(k))), k


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_device_hard_threshold_vs_oracle(dtype):
    from paper_2402_13781_b200 import sparsim as S
    acc = np.random.default_rng(3).laplace(size=11_200_000).astype(dtype)
    a = _dev(acc, dtype)
    for d in (0.0, 1e-3, 2.5, 4.605170185988091, 30.0):
        got = S.hard_threshold_select(a, d).cpu().numpy().astype(np.int64)
        assert np.array_equal(got, O.hard_threshold_select_np(acc, d)), d


@pytest.mark.gpu
def test_device_baselines_edge_cases():
    import torch
    from paper_2402_13781_b200 import sparsim as S
    empty = torch.empty(0, device="cuda:0")
    assert S.hard_threshold_select(empty, 0.5).numel() == 0
    with pytest.raises(S.InvalidArgument, match="topk_select: k out of range"):
        S.topk_select(empty, 1)
    two = _dev([1.0, 2.0], np.float32)
    with pytest.raises(S.InvalidArgument, match="topk_select: k out of range"):
        S.topk_select(two, 0)
    with pytest.raises(S.InvalidArgument, match="topk_select: k out of range"):
        S.topk_select(two, 3)
    with pytest.raises(S.InvalidArgument):
        S.topk_select(torch.zeros(4, dtype=torch.int32, device="cuda:0"), 1)
    assert S.topk_select(two, 1).cpu().tolist() == [1]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_device_baselines_unaligned_view(dtype):
    # a tensor view that is not 16-byte aligned takes the scalar-load path
    import torch
    from paper_2402_13781_b200 import sparsim as S
    base = np.random.default_rng(5).laplace(size=300_001).astype(dtype)
    view = torch.tensor(base, device="cuda:0")[1:]
    assert view.data_ptr() % 16 != 0
    got = S.hard_threshold_select(view, 1.5).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, O.hard_threshold_select_np(base[1:], 1.5))
    got = S.topk_select(view, 3001).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, O.topk_select_np(base[1:], 3001))


@pytest.mark.gpu
def test_device_baselines_follow_the_tensor_device():
    # acc on cuda:1 while the current device is cuda:0
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    from paper_2402_13781_b200 import sparsim as S
    acc = np.random.default_rng(6).laplace(size=100_000).astype(np.float32)
    torch.cuda.set_device(0)
    t = torch.tensor(acc, device="cuda:1")
    got = S.hard_threshold_select(t, 2.0).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, O.hard_threshold_select_np(acc, 2.0))


@pytest.mark.gpu
def test_device_quantile_unaligned_input():
    # K8 falls back to scalar loads for a vector that is not 16-byte aligned
    import torch
    from paper_2402_13781_b200 import sparsim as S
    base = np.random.default_rng(9).laplace(size=100_003).astype(np.float32)
    t = torch.tensor(base, device="cuda:0")[1:]
    mags = np.abs(base[1:].astype(np.float64))
    m = mags.shape[0]
    pos = min(m - 1, int(np.floor((1 - 0.01) * m)))
    want = np.partition(mags, pos)[pos]
    assert S.initial_threshold_device(t.data_ptr(), m, 0.01, "f32") == want
