"""CPU: the oracle AND the product's host-side C ABI against the reference's
golden fixtures (tests/golden/reference_golden.json, produced from the
unmodified reference by tests/golden/make_golden.py).

These run without a GPU and without /root/reference.
"""
import ctypes as C
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2402_13781_b200 import _abi as A
from paper_2402_13781_b200 import sparsim as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def cfg_from(d):
    c = A.exd_config()
    for k, v in d.items():
        setattr(c, k, v)
    return c


def mk_topo(sz, parts):
    t = A.exd_topology()
    t.n, t.sz_blk = len(parts), sz
    pos = 0
    for i, b in enumerate(parts):
        t.blk_part[i], t.blk_pos[i] = b, pos
        pos += b
    return t


# ---------------------------------------------------------------- config ----
@pytest.mark.parametrize("impl", ["oracle", "product"])
def test_validate_matches_reference(impl):
    for case in GOLD["config"]:
        c = cfg_from(case["in"])
        o = A.exd_config()
        if impl == "oracle":
            rc = O.orc().orc_validate(C.byref(c), C.byref(o))
            msg = O.orc().orc_last_error().decode()
        else:
            from paper_2402_13781_b200._lib import lib
            rc = lib().exd_validate(C.byref(c), C.byref(o))
            msg = lib().exd_last_error().decode()
        assert rc == case["rc"], case
        if rc == 0:
            assert o.k == case["k"]
        else:
            assert msg == case["msg"]


def test_validate_python_mirror_raises_invalid_argument():
    with pytest.raises(S.InvalidArgument, match="^n_b < n\\*min_blk$"):
        S.validate(S.SparsifierConfig(n=4, n_g=64, n_b=2, d=0.5, min_blk=1))
    with pytest.raises(ValueError, match="^k < n$"):
        S.validate(S.SparsifierConfig(n=2, n_g=400, n_b=2, d=0.0025, min_blk=1))
    assert S.validate(S.SparsifierConfig(n=2, n_g=1000, n_b=2, d=0.0015, min_blk=1)).k == 2


# -------------------------------------------------------------- topology ----
@pytest.mark.parametrize("impl", ["oracle", "product"])
def test_build_topology_matches_reference(impl):
    from paper_2402_13781_b200._lib import lib
    for case in GOLD["topology"]:
        ng, nb, n, mb = case["args"]
        t = A.exd_topology()
        w = C.create_string_buffer(256)
        if impl == "oracle":
            rc = O.orc().orc_build_topology(ng, nb, n, mb, C.byref(t), w, 256)
        else:
            rc = lib().exd_build_topology(ng, nb, n, mb, C.byref(t), w, 256)
        assert rc == case["rc"], case["args"]
        if rc:
            msg = (O.orc().orc_last_error() if impl == "oracle" else lib().exd_last_error()).decode()
            assert msg == case["msg"]
            continue
        assert t.sz_blk == case["topo"]["sz_blk"]
        assert t.parts() == case["topo"]["blk_part"]
        assert t.pos() == case["topo"]["blk_pos"]
        assert w.value.decode() == case["warning"]
        for p, (st, end) in enumerate(case["ranges"]):
            a, b = C.c_int64(), C.c_int64()
            if impl == "oracle":
                O.orc().orc_partition_range(C.byref(t), p, ng, C.byref(a), C.byref(b))
            else:
                assert lib().exd_partition_range(C.byref(t), p, ng, C.byref(a), C.byref(b)) == 0
            assert (a.value, b.value) == (st, end)


# ------------------------------------------------------------- allocator ----
@pytest.mark.parametrize("impl", ["oracle", "product"])
def test_rotate_adjust_allocate_match_reference(impl):
    from paper_2402_13781_b200._lib import lib
    L = O.orc() if impl == "oracle" else lib()
    rot = L.orc_rotate if impl == "oracle" else L.exd_rotate_to_partition_order
    adj = L.orc_adjust if impl == "oracle" else L.exd_adjust_topology
    alc = L.orc_allocate if impl == "oracle" else L.exd_allocate_partition
    for c in GOLD["rotate"]:
        o = (C.c_int64 * c["n"])()
        rot((C.c_int64 * c["n"])(*c["k_rank"]), c["t"], c["n"], o)
        assert list(o) == c["out"], c
    for c in GOLD["adjust"]:
        t = mk_topo(c["sz_blk"], c["blk_part"])
        k = (C.c_int64 * len(c["k"]))(*c["k"])
        mv, sk = C.c_int32(), C.c_int32()
        adj(C.byref(t), k, c["alpha"], c["blk_move"], c["min_blk"], c["n_g"], C.byref(mv), C.byref(sk))
        assert t.parts() == c["out_topo"]["blk_part"] and t.pos() == c["out_topo"]["blk_pos"], c
        assert list(k) == c["out_k"] and (mv.value, sk.value) == (c["moves"], c["skips"]), c
    for c in GOLD["allocate"]:
        t = mk_topo(c["sz_blk"], c["blk_part"])
        p, st, end = C.c_int32(), C.c_int64(), C.c_int64()
        alc(C.byref(t), c["t"], c["rank"], c["n_g"], C.byref(p), C.byref(st), C.byref(end))
        assert p.value == c["partition"] and [st.value, end.value] == c["range"], c


def test_python_mirror_known_answers():
    # test_allocator.cpp:73-89 through the Python mirror of the reference API
    topo = S.PartitionTopology(100, [4, 4], [0, 4])
    k = [30, 10]
    stats = S.adjust_topology(topo, k, 1.25, 1, 1, 800)
    assert topo.blk_part == [3, 5] and topo.blk_pos == [0, 3] and k == [25, 15]
    assert (stats.moves, stats.skips) == (1, 0)
    assert S.rotate_to_partition_order([101, 202, 303], 0, 3) == [202, 303, 101]
    a = S.allocate_partition(S.PartitionTopology(30, [1, 1], [0, 1]), 0, 1, 70)
    assert (a.partition, a.range.st, a.range.end) == (1, 30, 70)
    w = []
    t = S.build_topology(64, 4, 2, 1, warning=w)
    assert t.sz_blk == 16 and w
    with pytest.raises(S.InvalidArgument):
        S.build_topology(4096, 8, 4, 3)
    g = S.gather_stats([3, 1])
    assert (g.k_prime, g.m_t, g.c_t, g.f_t) == (4, 3, 4, 1.5)


# ------------------------------------------------------------- threshold ----
@pytest.mark.parametrize("impl", ["oracle", "product"])
def test_scale_threshold_bit_exact(impl):
    from paper_2402_13781_b200._lib import lib
    f = O.orc().orc_scale_threshold if impl == "oracle" else lib().exd_scale_threshold
    for c in GOLD["scale_threshold"]:
        assert f(c["k"], c["k_prime"], c["delta"], c["beta"], c["gamma"]) == c["out"], c


def test_initial_threshold_oracle():
    for c in GOLD["initial_threshold"]:
        a = np.array(c["mags"], dtype=np.float64)
        o = C.c_double()
        assert O.orc().orc_initial_threshold(a.ctypes.data_as(O.PD), len(a), c["d"], C.byref(o)) == 0
        assert o.value == c["out"]


# ----------------------------------------------------------- collectives ----
@pytest.mark.parametrize("impl", ["oracle", "product"])
def test_gather_accounting(impl):
    from paper_2402_13781_b200._lib import lib
    for c in GOLD["gather"]:
        if c["rc"]:
            continue
        counts = [len(x) for x in c["lists"]]
        st = A.exd_gather_stats()
        arr = (C.c_int64 * len(counts))(*counts)
        if impl == "oracle":
            O.orc().orc_gather_stats(arr, len(counts), C.byref(st))
        else:
            assert lib().exd_gather_stats_of(arr, len(counts), C.byref(st)) == 0
        assert (st.k_prime, st.m_t, st.c_t, st.f_t) == (c["k_prime"], c["m_t"], c["c_t"], c["f_t"])


# -------------------------------------------------------------- generator ---
def test_oracle_generator_matches_reference():
    for c in GOLD["generator"]:
        spec = O.stream_spec(**c["spec"])
        g = O.synthetic_gradient_orc(spec, c["t"], c["rank"])
        assert hashlib.sha256(g.tobytes()).hexdigest() == c["sha256_f64"], c["spec"]


# ----------------------------------------------------------------- engine ---
def test_oracle_engine_trace_row():
    tr = GOLD["engine_trace"]
    for dtype in (np.float64,):
        eng = O.OracleEngine(cfg_from(tr["config"]), dtype)
        rec = A.record_dict(eng.step([np.array(g) for g in tr["grads"]]))
        assert rec == tr["record"]
        for r in range(2):
            assert eng.x(r).tolist() == tr["x"][r]
            assert eng.e(r).tolist() == tr["e"][r]
        assert eng.state(0).delta == tr["delta"]
        assert eng.union().tolist() == tr["union"]


@pytest.mark.parametrize("ti", range(4))
def test_oracle_f64_reproduces_reference_trajectories(ti):
    tr = GOLD["trajectories"][ti]
    cfg = cfg_from(tr["config"])
    spec = O.stream_spec(**tr["stream"])
    eng = O.OracleEngine(cfg, np.float64)
    for t, row in enumerate(tr["rows"]):
        gs = [O.synthetic_gradient_orc(spec, t, r).astype(np.float32).astype(np.float64)
              for r in range(cfg.n)]
        rec = A.record_dict(eng.step(gs))
        assert rec == row["record"], t
        assert eng.union().tolist() == row["union"], t
        st = eng.state(0)
        assert st.delta == row["delta_after"]
        assert st.topology.parts() == row["topo_after"]["blk_part"]
    for r in range(cfg.n):
        assert hashlib.sha256(eng.x(r).tobytes()).hexdigest() == tr["x_sha256"][r]
        assert hashlib.sha256(eng.e(r).tobytes()).hexdigest() == tr["e_sha256"][r]


# ----------------------------------------------------------------- ledger ---
def test_format_csv_matches_reference_bytes():
    """runner.cpp:55-80 through the product's exd_format_csv."""
    tr = GOLD["trajectories"][GOLD["csv"]["trajectory"]]
    recs = [S.IterationRecord(**r["record"]) for r in tr["rows"]]
    assert S.format_csv(recs) == GOLD["csv"]["text"]
    assert S.format_csv([]) == "t,k_prime,density,eps,m_t,C_t,f_t,global_err,delta,loss\n"


def test_summarize_matches_reference():
    tr = GOLD["trajectories"][1]
    dicts = [r["record"] for r in tr["rows"]]
    s = S.summarize([S.IterationRecord(**d) for d in dicts])
    n = len(dicts)
    assert s["iterations"] == n
    acc = 0.0  # sequential, like runner.cpp:94 (Python's sum() is compensated)
    for d in dicts:
        acc += d["density"]
    assert s["mean_density"] == acc / n
    assert s["final_delta"] == dicts[-1]["delta"]
    assert s["adjust_moves"] == sum(d["adjust_moves"] for d in dicts)
    if O.ref_available():
        arr = O.records_array(dicts)
        d6 = (C.c_double * 6)()
        i5 = (C.c_int64 * 5)()
        O.ref().ref_summarize(arr, n, d6, i5)
        assert [s["mean_density"], s["mean_f"], s["mean_eps"], s["mean_idle_workers"],
                s["final_delta"], s["final_global_err"]] == list(d6)
        assert [s["iterations"], s["duplicates"], s["adjust_moves"], s["adjust_skips"],
                s["cap_hits"]] == list(i5)
