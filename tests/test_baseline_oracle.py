"""CPU: the numpy restatement of the baseline-sparsifier Engine runs
(oracle.BaselineOracle) is pinned bit-exact against the unmodified reference
(oracle/_ref, sparsim::Engine with SparsifierKind TopK / CLTk / HardThreshold)
in fp64: records, union, x and e."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("kind,fixed", [("topk", 0.0), ("cltk", 0.0), ("hardthreshold", 1.7)])
@pytest.mark.parametrize("n", [1, 3])
def test_baseline_oracle_matches_reference(kind, fixed, n):
    n_g, d = 20_011, 0.01
    cfg = O.make_config(n=n, n_g=n_g, n_b=16, d=d, seed=3)
    ref = O.RefEngine(cfg, O.make_options(sparsifier=O.BaselineOracle.KINDS[kind],
                                          fixed_delta=fixed, verify_conservation=1), pool=n)
    k = int(round(d * n_g))
    orc = O.BaselineOracle(n, n_g, k, kind, fixed, dtype=np.float64)
    spec = O.stream_spec(n_g, O.skew_segments(n_g), seed=3)
    for t in range(12):
        grads = [O.synthetic_gradient_orc(spec, t, r) for r in range(n)]
        rrec = O.A.record_dict(ref.step(grads, capture=True))
        orec = orc.step(grads)
        for f, v in orec.items():
            if f == "global_err":
                assert abs(rrec[f] - v) <= 1e-12 * max(abs(v), 1e-300), (t, f)
            else:
                assert rrec[f] == v, (t, f, rrec[f], v)
        assert np.array_equal(ref.union(), orc.last_union), t
    for r in range(n):
        assert np.array_equal(ref.x(r), orc.x[r]) and np.array_equal(ref.e(r), orc.e[r])
