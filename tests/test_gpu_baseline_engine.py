"""GPU: Engine runs of the baseline sparsifiers: Top-k,
CLT-k and hard threshold through the device engine (engine.cpp:163-204,
274-350), with the deduplicating union (collectives.cpp:47-55).

  * fp32: bit-exact against the numpy restatement oracle.BaselineOracle
    (itself pinned against the unmodified reference, test_baseline_oracle.py);
  * fp64: bit-exact against the unmodified reference (oracle/_ref);
  * acceptance C1 (build-up elimination, acceptance_main.cpp:157-180) and C3
    (hard-threshold failure mode, :201-232) on the reference's main run.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2402_13781_b200 import sparsim as S

pytestmark = pytest.mark.gpu

KINDS = [("topk", 0.0), ("cltk", 0.0), ("hardthreshold", 2.2)]


def _grads(src, t, n, bufs, dtype, stream):
    import torch
    for r in range(n):
        src.gradient(t, r, bufs[r], dtype, stream)
    torch.cuda.synchronize()
    return [b.cpu().numpy() for b in bufs]


def _check(rec, orec, ctx):
    o = orec if isinstance(orec, dict) else O.A.record_dict(orec)
    for f in ("t", "k_prime", "density", "eps", "m_t", "c_t", "f_t", "delta", "duplicates",
              "union_count", "adjust_moves", "adjust_skips", "cap_hits", "idle_workers"):
        assert getattr(rec, f) == o[f], (ctx, f, getattr(rec, f), o[f])
    assert rec.k_rank == list(o["k_rank"]), ctx
    assert abs(rec.global_err - o["global_err"]) <= 1e-6 * max(abs(o["global_err"]), 1e-300), ctx


@pytest.mark.parametrize("kind,fixed", KINDS, ids=[k for k, _ in KINDS])
@pytest.mark.parametrize("n", [1, 3, 8])
def test_baseline_engine_fp32_bit_exact_vs_oracle(kind, fixed, n):
    import torch
    n_g, d = 300_007, 0.004
    cfg = S.SparsifierConfig(n=n, n_g=n_g, n_b=64, d=d, seed=9)
    eng = S.Engine(cfg, S.EngineOptions(sparsifier=kind, fixed_delta=fixed,
                                        verify_conservation=True))
    k = S.validate(cfg).k
    orc = O.BaselineOracle(n, n_g, k, kind, fixed, dtype=np.float32)
    src = S.SyntheticStream(S.StreamSpec(n_g=n_g, segments=O.skew_segments(n_g), seed=9))
    bufs = [torch.empty(n_g, device="cuda") for _ in range(n)]
    for t in range(15):
        host = _grads(src, t, n, bufs, "f32", eng.stream())
        rec = eng.step(bufs)
        orec = orc.step(host)
        _check(rec, orec, f"t={t}")
        assert np.array_equal(eng.idx_global(0).astype(np.int64), orc.last_union), t
        np.testing.assert_array_equal(eng.reduced(0), orc.last_sum)
    for w in range(n):
        assert np.array_equal(eng.x(w), orc.x[w]) and np.array_equal(eng.e(w), orc.e[w]), w
        assert eng.k_t(w) == orc.k_t
    eng.close()


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("kind,fixed", KINDS, ids=[k for k, _ in KINDS])
def test_baseline_engine_fp64_bit_exact_vs_reference(kind, fixed):
    import torch
    n, n_g, d = 3, 200_003, 0.005
    kw = dict(n=n, n_g=n_g, n_b=48, d=d, seed=4)
    eng = S.Engine(S.SparsifierConfig(**kw), S.EngineOptions(sparsifier=kind, fixed_delta=fixed,
                                                             dtype="f64"))
    ref = O.RefEngine(O.make_config(**kw), O.make_options(
        sparsifier=O.BaselineOracle.KINDS[kind], fixed_delta=fixed), pool=n)
    src = S.SyntheticStream(S.StreamSpec(n_g=n_g, seed=4))
    bufs = [torch.empty(n_g, dtype=torch.float64, device="cuda") for _ in range(n)]
    for t in range(10):
        host = _grads(src, t, n, bufs, "f64", eng.stream())
        rec = eng.step(bufs)
        orec = ref.step(host, capture=True)
        _check(rec, orec, f"t={t}")
        assert np.array_equal(eng.idx_global(0).astype(np.int64), ref.union()), t
    for w in range(n):
        assert np.array_equal(eng.x(w), ref.x(w)) and np.array_equal(eng.e(w), ref.e(w)), w
        assert eng.delta(w) == ref.state(w).delta
    eng.close()


MAIN = dict(n=8, n_g=1_000_000, d=0.001, seed=7)


def _main_run(kind, fixed=0.0, iters=1000, decay_step=None):
    import torch
    cfg = S.SparsifierConfig(**MAIN)
    eng = S.Engine(cfg, S.EngineOptions(sparsifier=kind, fixed_delta=fixed,
                                        verify_replication=False, verify_conservation=True))
    src = S.SyntheticStream(S.StreamSpec(n_g=cfg.n_g, seed=cfg.seed, decay_step=decay_step))
    bufs = [torch.empty(cfg.n_g, device="cuda") for _ in range(cfg.n)]
    recs = eng.run(iters, src, bufs)
    eng.close()
    return recs


def test_c1_build_up_elimination():
    """acceptance_main.cpp:157-180: ExDyna and CLT-k never select an index
    twice; Top-k's union lies in (k, 8k] on >= 95% of the iterations."""
    k = S.validate(S.SparsifierConfig(**MAIN)).k
    ex = _main_run("exdyna")
    clt = _main_run("cltk")
    top = _main_run("topk")
    assert sum(r.duplicates for r in ex) == 0
    assert sum(r.duplicates for r in clt) == 0
    frac = np.mean([k < r.union_count <= 8 * k for r in top])
    assert frac >= 0.95, frac


def test_c3_hard_threshold_failure_mode():
    """acceptance_main.cpp:201-232: a threshold fixed at half ExDyna's
    converged delta over-selects (mean density > 2d), and after the gradient
    scale drops 10x at t = 500 the hard threshold under-selects."""
    ex = _main_run("exdyna")
    fixed = 0.5 * float(np.mean([r.delta for r in ex[-100:]]))
    d = MAIN["d"]
    stat = _main_run("hardthreshold", fixed)
    mean = float(np.mean([r.density for r in stat]))
    stepped = _main_run("hardthreshold", fixed, decay_step=500)
    pre = float(np.mean([r.density for r in stepped[:500]]))
    post = float(np.mean([r.density for r in stepped[500:]]))
    assert mean > 2 * d and post < pre, (mean / d, pre / d, post / d)
