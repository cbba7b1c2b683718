"""GPU: the BASELINE.json configurations at their full sizes.

  * SE-18  (n_g = 11.3M, d = 0.01): the 200-iteration threshold-scaling
           trajectory, bit-exact vs the fp32 oracle, and (fp64 mode) vs the
           unmodified reference.
  * GN     (n_g = 6.2M, d in {0.001, 0.01}, skewed magnitudes, n = 8):
           bit-exact vs the oracle, and dynamic partitioning lowers the padding
           ratio f_t against static partitions (acceptance C4,
           acceptance_main.cpp:234-248).
  * R18    (n_g = 11.2M, d = 0.01, n = 8): bit-exact steps + structural
           properties (ascending union, exclusive ownership, conservation).
  * sweep  (configs[4], n_g 10M / 100M / 1B): multi-step trajectories
           bit-exact vs the fp32 oracle (records, selections, per-block
           counts, delta, topology, and x / e at the end), plus size-
           independent properties of one step checked on the device.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2402_13781_b200 import sparsim as S

from pairing import Pair, check_record

pytestmark = pytest.mark.gpu


def _pinned(**kw):
    base = dict(n_b=256, alpha=1.25, beta=1.25, gamma=0.02, blk_move=1, min_blk=2, eta=1.0)
    base.update(kw)
    return base


def test_se18_200_iteration_threshold_trajectory_fp32():
    kw = _pinned(n=2, n_g=11_300_000, d=0.01, seed=7)
    p = Pair(kw, "f32", verify_replication=False)
    deltas = []
    for t in range(200):
        rec, orec = p.step(t)
        check_record(rec, orec, ctx=f"t={t}")
        deltas.append(rec.delta)
        if t % 50 == 49:
            p.compare_selection(ctx=f"t={t}")
            p.compare_state(ctx=f"t={t}", vectors=(t == 199))
    # the controller actually moved: the trajectory is not a constant
    assert len(set(deltas)) > 100


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_se18_200_iteration_trajectory_fp64_vs_unmodified_reference():
    kw = _pinned(n=2, n_g=11_300_000, d=0.01, seed=7)
    p = Pair(kw, "f64", checker="reference", verify_replication=False)
    for t in range(200):
        host = p.gradients(t)
        rec = p.eng.step(p.bufs)
        orec = p.chk.step([h.astype(np.float64) for h in host], capture=False)
        check_record(rec, orec, ctx=f"t={t}", err_rtol=1e-12)
    p.compare_state(ctx="end", vectors=True)


@pytest.mark.parametrize("d", [0.001, 0.01])
def test_googlenet_skew_n8_bit_exact(d):
    kw = _pinned(n=8, n_g=6_200_000, d=d, seed=1)
    p = Pair(kw, "f32", segments=O.skew_segments(6_200_000), verify_replication=True)
    for t in range(40):
        rec, orec = p.step(t)
        check_record(rec, orec, ctx=f"t={t}")
        if t % 10 == 9:
            p.compare_selection(ctx=f"t={t}")
    p.compare_state(ctx="end")


def test_googlenet_dynamic_partitions_reduce_padding():
    """acceptance C4: skewed stream, dynamic f_t < static f_t."""
    import torch
    n_g, n = 6_200_000, 8
    segs = O.skew_segments(n_g)
    src = S.SyntheticStream(S.StreamSpec(n_g=n_g, segments=segs, seed=1))
    res = {}
    for static in (False, True):
        eng = S.Engine(S.SparsifierConfig(**_pinned(n=n, n_g=n_g, d=0.01, seed=1)),
                       S.EngineOptions(static_partitions=static, verify_replication=False))
        bufs = [torch.empty(n_g, device="cuda") for _ in range(n)]
        fts = []
        for t in range(160):
            for r in range(n):
                src.gradient(t, r, bufs[r], "f32", eng.stream())
            rec = eng.step(bufs)
            if t >= 60:
                fts.append(rec.f_t)
            assert rec.duplicates == 0
        res[static] = float(np.mean(fts))
    assert res[False] < res[True], res


def test_r18_n8_full_size_bit_exact_and_structural():
    kw = _pinned(n=8, n_g=11_200_000, d=0.01, seed=7)
    p = Pair(kw, "f32", verify_replication=True)
    for t in range(6):
        e_before = [p.eng.e(w) for w in range(8)] if t == 5 else None
        rec, orec = p.step(t)
        check_record(rec, orec, ctx=f"t={t}")
        p.compare_selection(ctx=f"t={t}")
    # structural properties of the last step
    u = p.eng.idx_global(0).astype(np.int64)
    assert np.all(np.diff(u) > 0)  # strictly ascending union
    sels = [p.eng.selection(w).astype(np.int64) for w in range(8)]
    assert sum(len(s) for s in sels) == rec.k_prime == len(u)
    assert np.array_equal(np.sort(np.concatenate(sels)), u)  # exclusive ownership, no dups
    st = p.eng.state(0)
    for w in range(8):  # every selection lies inside its owner's partition
        s = p.eng.state(w)
        if len(sels[w]):
            assert s.st <= sels[w][0] and sels[w][-1] < s.end
    # error-feedback mass conservation at the union (selector test :64-86):
    # contribution (all-reduced) == sum over workers of acc at the union
    host = [b.cpu().numpy() for b in p.bufs]
    acc = [(e_before[w] + host[w]).astype(np.float32) for w in range(8)]
    g = p.eng.reduced(0)
    s = acc[0][u]
    for w in range(1, 8):
        s = s + acc[w][u]
    np.testing.assert_array_equal(g, s)
    for w in range(8):
        assert not np.any(p.eng.e(w)[u])
    assert st.t == 6


def _host_bytes_available():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


SWEEP_CELLS = [
    # n_g, d, n, steps
    (10_000_000, 0.001, 1, 30),
    (10_000_000, 0.1, 2, 30),
    (100_000_000, 0.01, 1, 30),
    (100_000_000, 0.001, 2, 20),
    (100_000_000, 0.1, 1, 12),
    (1_000_000_000, 0.01, 1, 3),
]


@pytest.mark.parametrize("n_g,d,n,steps", SWEEP_CELLS,
                         ids=lambda v: str(v))
def test_sweep_multi_step_bit_exact_vs_oracle(n_g, d, n, steps):
    """configs[4] cells: the whole trajectory (t = 0 quantile, adjust, delta
    scaling) equals the fp32 restatement of engine.cpp:274-350 step by step."""
    import torch
    free, _ = torch.cuda.mem_get_info(0)
    if free < 40 * n * n_g:
        pytest.skip("not enough device memory")
    if _host_bytes_available() < 40 * n * n_g:
        pytest.skip("not enough host memory for the oracle")
    kw = _pinned(n=n, n_g=n_g, d=d, seed=7)
    p = Pair(kw, "f32", verify_replication=False)
    for t in range(steps):
        rec, orec = p.step(t)
        check_record(rec, orec, ctx=f"t={t}")
        if t % 10 == 9 or t == steps - 1:
            p.compare_selection(ctx=f"t={t}")
    p.compare_state(ctx="end", vectors=True)
    assert rec.t == steps - 1


@pytest.mark.parametrize("n_g,d", [(1_000_000, 0.1), (100_000_000, 0.001), (1_000_000_000, 0.01)])
def test_sweep_one_step_properties(n_g, d):
    """Size-independent properties of a single step from e = 0 with a given
    delta0: selection == {|g| >= delta0}, residual keeps the rest, x = -g at
    the selection, k' matches a device count; checked with device reductions."""
    import torch
    if torch.cuda.get_device_properties(0).total_memory < 40 * n_g:
        pytest.skip("not enough device memory")
    delta0 = 1.5
    eng = S.Engine(S.SparsifierConfig(n=1, n_g=n_g, n_b=256, d=d, delta0=delta0, seed=3),
                   S.EngineOptions(verify_replication=False))
    g = torch.empty(n_g, device="cuda")
    S.SyntheticStream(S.StreamSpec(n_g=n_g, seed=3)).gradient(0, 0, g, "f32", eng.stream())
    torch.cuda.synchronize()
    rec = eng.step([g])
    sel = g.abs() >= delta0
    assert rec.k_prime == int(sel.sum())
    assert rec.m_t == rec.k_prime and rec.c_t == 0 and rec.f_t == 1.0
    assert rec.delta == delta0
    del sel
    torch.cuda.empty_cache()
    idx = eng.device_view(0, "idx_global").long()
    assert bool((idx[1:] > idx[:-1]).all())
    assert bool((g[idx].abs() >= delta0).all())
    e = eng.device_view(0, "e")
    x = eng.device_view(0, "x")
    for lo in range(0, n_g, 1 << 27):  # windows keep the temporaries small at 1B
        hi = min(n_g, lo + (1 << 27))
        gw = g[lo:hi]
        selw = gw.abs() >= delta0
        assert torch.equal(e[lo:hi], torch.where(selw, torch.zeros_like(gw), gw))
        assert torch.equal(x[lo:hi], torch.where(selw, -gw, torch.zeros_like(gw)))
