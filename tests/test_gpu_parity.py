"""GPU parity: the B200 path against the oracle (fp32 restatement, bit-exact)
and against the unmodified reference (fp64 mode, bit-exact), through the C ABI.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2402_13781_b200 import sparsim as S

from pairing import Pair, check_record

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "the -m gpu suite needs a B200"
    yield


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_hand_traced_row(dtype):
    """test_engine.cpp:79-131 on the device."""
    import torch
    tr = GOLD["engine_trace"]
    c = tr["config"]
    cfg = S.SparsifierConfig(n=c["n"], n_g=c["n_g"], n_b=c["n_b"], d=c["d"], min_blk=c["min_blk"],
                             delta0=c["delta0"], eta=c["eta"], beta=c["beta"], gamma=c["gamma"])
    eng = S.Engine(cfg, S.EngineOptions(dtype=dtype))
    td = torch.float64 if dtype == "f64" else torch.float32
    grads = [torch.tensor(g, dtype=td, device="cuda") for g in tr["grads"]]
    rec = eng.step(grads)
    want = tr["record"]
    assert (rec.t, rec.k_prime, rec.m_t, rec.c_t, rec.union_count) == (0, 3, 2, 2, 3)
    assert rec.k_rank == [2, 1] and rec.delta == 0.5 and rec.global_err == 0.0
    assert rec.f_t == want["f_t"] and rec.density == want["density"] and rec.eps == want["eps"]
    assert eng.idx_global().tolist() == tr["union"]
    if dtype == "f64":
        for r in range(2):
            assert eng.x(r).tolist() == tr["x"][r]
            assert eng.e(r).tolist() == tr["e"][r]
    else:
        for r in range(2):
            np.testing.assert_array_equal(eng.e(r), np.array(tr["e"][r], dtype=np.float32))
    assert eng.delta(0) == tr["delta"] and eng.k_t(0) == [2, 1]
    # the cyclic allocation hands worker 0 the other partition at t=1
    a = S.allocate_partition(eng.topology(0), 1, 0, 8)
    assert (a.range.st, a.range.end) == (4, 8)


CONFIGS = [
    # n, n_g, n_b, d, extra
    dict(n=1, n_g=50_000, n_b=16, d=0.01, seed=3),
    dict(n=2, n_g=100_000, n_b=32, d=0.01, seed=4),
    dict(n=3, n_g=77_777, n_b=24, d=0.02, seed=5),
    dict(n=4, n_g=200_003, n_b=64, d=0.005, seed=6, beta=1.05),
    dict(n=8, n_g=300_000, n_b=256, d=0.01, seed=7),
    dict(n=2, n_g=4097, n_b=16, d=0.05, seed=8, eta=0.7, delta0=0.8),
    dict(n=5, n_g=33_333, n_b=40, d=0.03, seed=9, alpha=1.1, blk_move=2, min_blk=3),
    dict(n=2, n_g=9, n_b=2, d=0.5, seed=10, min_blk=1),
    dict(n=1, n_g=8, n_b=1, d=0.5, seed=11, min_blk=1),
]


@pytest.mark.parametrize("kw", CONFIGS, ids=lambda k: f"n{k['n']}_g{k['n_g']}")
@pytest.mark.parametrize("skew", [False, True])
def test_fp32_bit_exact_vs_oracle(kw, skew):
    segs = O.skew_segments(kw["n_g"]) if skew and kw["n_g"] >= 64 else None
    p = Pair(kw, "f32", segments=segs)
    for t in range(25):
        rec, orec = p.step(t)
        check_record(rec, orec, ctx=f"t={t}")
        p.compare_selection(ctx=f"t={t}")
        if t % 6 == 0 or t == 24:
            p.compare_state(ctx=f"t={t}")


@pytest.mark.parametrize("kw", CONFIGS[:6], ids=lambda k: f"n{k['n']}_g{k['n_g']}")
def test_fp64_bit_exact_vs_reference(kw):
    checker = "reference" if O.ref_available() else "oracle"
    p = Pair(kw, "f64", checker=checker)
    for t in range(20):
        rec, orec = p.step(t)
        check_record(rec, orec, ctx=f"t={t}")
        p.compare_selection(ctx=f"t={t}")
    p.compare_state(ctx="end")


@pytest.mark.parametrize("ti", range(4))
def test_fp64_reproduces_golden_reference_trajectory(ti):
    """The committed reference trajectories (no /root/reference needed)."""
    import torch
    tr = GOLD["trajectories"][ti]
    c = tr["config"]
    cfg = S.SparsifierConfig(n=c["n"], n_g=c["n_g"], n_b=c["n_b"], d=c["d"], seed=c["seed"],
                             delta0=c["delta0"] if c["has_delta0"] else None, alpha=c["alpha"],
                             beta=c["beta"], gamma=c["gamma"], blk_move=c["blk_move"],
                             min_blk=c["min_blk"], eta=c["eta"])
    eng = S.Engine(cfg, S.EngineOptions(dtype="f64"))
    spec = O.stream_spec(**tr["stream"])
    bufs = [torch.empty(c["n_g"], dtype=torch.float64, device="cuda") for _ in range(c["n"])]
    recs = []
    for t, row in enumerate(tr["rows"]):
        for r in range(c["n"]):
            g = O.synthetic_gradient_orc(spec, t, r).astype(np.float32).astype(np.float64)
            bufs[r].copy_(torch.from_numpy(g))
        torch.cuda.synchronize()
        rec = eng.step(bufs)
        recs.append(rec)
        want = row["record"]
        for f in ("k_prime", "m_t", "c_t", "f_t", "delta", "density", "eps", "adjust_moves",
                  "adjust_skips", "union_count"):
            assert getattr(rec, f) == want[f], (t, f)
        assert rec.k_rank == want["k_rank"]
        assert abs(rec.global_err - want["global_err"]) <= 1e-12 * max(want["global_err"], 1e-300)
        assert eng.idx_global().tolist() == row["union"], t
        assert eng.delta(0) == row["delta_after"]
        assert eng.topology(0).blk_part == row["topo_after"]["blk_part"]
    for r in range(c["n"]):
        assert hashlib.sha256(eng.x(r).tobytes()).hexdigest() == tr["x_sha256"][r]
        assert hashlib.sha256(eng.e(r).tobytes()).hexdigest() == tr["e_sha256"][r]
    if ti == GOLD["csv"]["trajectory"]:
        # the CSV ledger (runner.cpp:55-80) byte for byte, except global_err,
        # which the device reduces as a tree (<= 1e-12 relative in fp64 mode)
        def drop_err(text):
            return [",".join(l.split(",")[:7] + l.split(",")[8:]) for l in text.splitlines()]
        assert drop_err(S.format_csv(recs)) == drop_err(GOLD["csv"]["text"])


def test_static_partitions():
    p = Pair(dict(n=4, n_g=64_000, n_b=32, d=0.01, seed=12), "f32",
             segments=O.skew_segments(64_000), static=True)
    for t in range(15):
        rec, orec = p.step(t)
        check_record(rec, orec, ctx=f"t={t}")
        assert rec.adjust_moves == 0
    p.compare_state()


def test_lognormal_stream():
    p = Pair(dict(n=3, n_g=60_000, n_b=30, d=0.01, seed=13), "f32", distribution=1)
    for t in range(12):
        rec, orec = p.step(t)
        check_record(rec, orec, ctx=f"t={t}")
        p.compare_selection()
    p.compare_state()


def test_zero_gradients_select_nothing():
    import torch
    cfg = S.SparsifierConfig(n=2, n_g=10_000, n_b=8, d=0.01, delta0=0.5)
    eng = S.Engine(cfg)
    z = [torch.zeros(10_000, device="cuda") for _ in range(2)]
    for t in range(3):
        rec = eng.step(z)
        assert rec.k_prime == 0 and rec.m_t == 0 and rec.c_t == 0 and rec.f_t == 1.0
        assert rec.k_rank == [0, 0]
    # under the band: delta shrinks by gamma every step
    d = 0.5
    for _ in range(3):
        d = S.scale_threshold(100, 0, d, 1.25, 0.02)
    assert eng.delta() == d


def test_zero_gradients_auto_delta_floor():
    """engine.cpp:157: an all-zero first accumulation floors delta0 at 1e-300."""
    import torch
    eng = S.Engine(S.SparsifierConfig(n=1, n_g=5000, n_b=4, d=0.01))
    rec = eng.step([torch.zeros(5000, device="cuda")])
    assert rec.delta == 1e-300 and rec.k_prime == 0


def test_density_one_is_dense_sgd():
    """test_engine.cpp:228-264 with synthetic gradients: d=1 and a tiny delta
    select every non-zero coordinate; x follows dense SGD exactly."""
    import torch
    n, n_g = 2, 4096
    cfg = S.SparsifierConfig(n=n, n_g=n_g, n_b=4, d=1.0, delta0=1e-300, eta=0.1, seed=5)
    eng = S.Engine(cfg, S.EngineOptions(dtype="f64"))
    src = S.SyntheticStream(S.StreamSpec(n_g=n_g, seed=5))
    bufs = [torch.empty(n_g, dtype=torch.float64, device="cuda") for _ in range(n)]
    x = np.zeros(n_g)
    for t in range(30):
        for r in range(n):
            src.gradient(t, r, bufs[r], "f64", eng.stream())
        torch.cuda.synchronize()
        g = [b.cpu().numpy() for b in bufs]
        rec = eng.step(bufs)
        assert rec.k_prime == n_g
        s = 0.1 * g[0] + 0.1 * g[1]
        x = x - s / 2
        np.testing.assert_array_equal(eng.x(0), x)
        assert not np.any(eng.e(0))


def test_replication_divergence_raises():
    """test_engine.cpp:219-226: perturbing x on rank 1 aborts the next step."""
    p = Pair(dict(n=3, n_g=2048, n_b=12, d=0.01, seed=11), "f32")
    p.step(0)
    p.step(1)
    x = p.eng.x(1)
    x[3] += 1.0
    p.eng.write(1, "x", x)
    with pytest.raises(S.EngineError, match="replicated state diverged at iteration 2: rank 1 field x"):
        p.step(2)


def test_step_host_matches_device_step():
    import torch
    kw = dict(n=2, n_g=100_000, n_b=16, d=0.01, seed=21)
    a = S.Engine(S.SparsifierConfig(**kw))
    b = S.Engine(S.SparsifierConfig(**kw))
    src = S.SyntheticStream(S.StreamSpec(n_g=kw["n_g"], seed=21))
    bufs = [torch.empty(kw["n_g"], device="cuda") for _ in range(2)]
    for t in range(8):
        for r in range(2):
            src.gradient(t, r, bufs[r], "f32", a.stream())
        torch.cuda.synchronize()
        host = [x.cpu().numpy() for x in bufs]
        ra = a.step(bufs)
        rb = b.step_host(host)
        assert ra == rb
    np.testing.assert_array_equal(a.x(0), b.x(0))


def test_device_generator_matches_reference_stream():
    """SyntheticStream on the device vs the reference generator (workloads.cpp:62-85).
    The counter-based draws are bit-identical; only the device log1p/exp may
    differ from glibc in the last place."""
    import torch
    for c in GOLD["generator"]:
        spec_kw = c["spec"]
        spec = O.stream_spec(**spec_kw)
        want = O.synthetic_gradient_orc(spec, c["t"], c["rank"])
        assert hashlib.sha256(want.tobytes()).hexdigest() == c["sha256_f64"]
        src = S.SyntheticStream(S.StreamSpec(
            n_g=spec_kw["n_g"], segments=spec_kw.get("segments"), seed=spec_kw["seed"],
            distribution=spec_kw.get("distribution", 0), decay=spec_kw.get("decay", 1.0),
            decay_step=spec_kw.get("decay_step")))
        buf = torch.empty(spec_kw["n_g"], dtype=torch.float64, device="cuda")
        src.gradient(c["t"], c["rank"], buf, "f64")
        torch.cuda.synchronize()
        got = buf.cpu().numpy()
        rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-300)
        # device log1p/log/exp/cos vs glibc: a few ulp at most; most draws are
        # bit-identical (the path's parity tests feed the SAME buffers to both)
        assert rel.max() <= 2e-15, rel.max()
        assert np.mean(got == want) > 0.8


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_device_quantile_matches_nth_element(dtype):
    """threshold.cpp:37-47 (nth_element) vs the device radix select, incl. ties."""
    import torch
    rng = np.random.default_rng(7)
    td = torch.float64 if dtype == "f64" else torch.float32
    nd = np.float64 if dtype == "f64" else np.float32
    cases = [np.abs(rng.laplace(size=1_000_003)).astype(nd),
             np.repeat(np.array([2.5, 1.0, 3.0], dtype=nd), 1000),
             -np.abs(rng.normal(size=4097)).astype(nd),
             np.zeros(100, dtype=nd), np.array([7.0], dtype=nd)]
    for a in cases:
        for d in (0.001, 0.01, 0.25, 1.0):
            m = len(a)
            pos = min(m - 1, int(np.floor((1.0 - d) * m)))
            want = float(np.partition(np.abs(a).astype(np.float64), pos)[pos])
            buf = torch.from_numpy(a).to("cuda")
            got = S.initial_threshold_device(buf.data_ptr(), m, d, dtype)
            assert got == want, (m, d)


def test_kernel_stats_and_unsupported_options():
    import torch
    # engine.cpp:58-61
    with pytest.raises(S.InvalidArgument, match="fixed_delta out of range"):
        S.Engine(S.SparsifierConfig(n=2, n_g=1000, n_b=8, d=0.01),
                 S.EngineOptions(sparsifier="hardthreshold"))
    eng = S.Engine(S.SparsifierConfig(n=1, n_g=100_000, n_b=8, d=0.01),
                   S.EngineOptions(profile_kernels=True))
    g = torch.randn(100_000, device="cuda")
    for _ in range(3):
        eng.step([g])
    st = eng.kernel_stats()
    # t=0 without delta0: accumulate + select-only launches, then one fused launch per step
    assert st["select_launches"] == 4 and st["select_ms"] > 0 and st["steps"] == 3
    # t = 0: accumulate, K8 (init + 3 x (hist + pick) + out for fp32), set_delta,
    # select-only + finish; then stream + finish per step
    assert st["kernel_launches"] == 1 + 8 + 1 + 2 + 2 * 2
    # gradients must be 16-byte aligned, the right dtype and n_g long
    flat = torch.zeros(100_004, device="cuda")
    with pytest.raises(S.InvalidArgument, match="16-byte aligned"):
        eng.step([flat[1:100_001]])
    with pytest.raises(S.InvalidArgument, match="workload size"):
        eng.step([flat])
    with pytest.raises(S.InvalidArgument, match="dtype"):
        eng.step([flat[:100_000].double()])
    from paper_2402_13781_b200._lib import lib
    import ctypes as C
    rc = lib().exd_engine_step_async(eng.h, (C.c_void_p * 1)(flat.data_ptr() + 4))
    assert rc == S.A.EXD_EINVAL
    eng.step([flat[:100_000]])  # the engine is still usable


CAP_CONFIGS = [
    dict(n=1, n_g=40_000, n_b=8, d=0.02, seed=3, max_density_cap=0.006),
    dict(n=2, n_g=100_001, n_b=32, d=0.02, seed=4, max_density_cap=0.005),
    dict(n=3, n_g=60_000, n_b=24, d=0.05, seed=5, max_density_cap=0.01, beta=1.05),
]


@pytest.mark.parametrize("kw", CAP_CONFIGS, ids=lambda k: f"n{k['n']}")
@pytest.mark.parametrize("quantum", [None, 0.25])
def test_density_cap_fp32_vs_oracle(kw, quantum):
    """selector.cpp:44-61: cap hits, kept set (largest |acc|, lower index on
    ties), restored residuals and cap_hits in the ledger, bit-exact."""
    p = Pair(kw, "f32")
    hits = 0
    for t in range(15):
        rec, orec = p.step(t, quantum=quantum)
        check_record(rec, orec, ctx=f"t={t}")
        p.compare_selection(ctx=f"t={t}")
        hits += rec.cap_hits
    p.compare_state(ctx="end")
    assert hits > 0


@pytest.mark.parametrize("kw", CAP_CONFIGS[:2], ids=lambda k: f"n{k['n']}")
def test_density_cap_fp64_vs_reference(kw):
    checker = "reference" if O.ref_available() else "oracle"
    p = Pair(kw, "f64", checker=checker)
    for t in range(12):
        rec, orec = p.step(t)
        check_record(rec, orec, ctx=f"t={t}")
    p.compare_state(ctx="end")


@pytest.mark.parametrize("kw", [CONFIGS[0], CONFIGS[2], CAP_CONFIGS[1], CONFIGS[7]],
                         ids=lambda k: f"n{k['n']}_g{k['n_g']}")
def test_verify_conservation_holds(kw):
    """engine.cpp:221-249 on the device: every step's contributions equal the
    acc snapshot at the union, the union is cleared, nothing else moves."""
    p = Pair(kw, "f32", verify_conservation=True)
    for t in range(8):
        rec, orec = p.step(t)
        check_record(rec, orec, ctx=f"t={t}")
