"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the container that has /root/reference (oracle/_ref is built from it):

    python tests/golden/make_golden.py

Every fixture is produced by calling the reference's own functions / Engine
through oracle/ref_shim.cpp; the known-answer inputs are those of the
reference's unit tests (test_partition.cpp, test_allocator.cpp,
test_threshold.cpp, test_collectives.cpp, test_config.cpp, test_engine.cpp)
plus seeded random cases. The GPU box has no /root/reference: tests read these
files instead.
"""
import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2402_13781_b200 import _abi as A  # noqa: E402


def cfg_dict(c):
    return {f: getattr(c, f) for f, _ in A.exd_config._fields_}


def topo_dict(t):
    return {"sz_blk": t.sz_blk, "blk_part": t.parts(), "blk_pos": t.pos()}


def mk_topo(sz, parts):
    t = A.exd_topology()
    t.n, t.sz_blk = len(parts), sz
    pos = 0
    for i, b in enumerate(parts):
        t.blk_part[i], t.blk_pos[i] = b, pos
        pos += b
    return t


def main():
    R = O.ref()
    rng = np.random.default_rng(2402_13781)
    out = {}

    # --- config (test_config.cpp:37-110) -----------------------------------
    cases = []
    base = dict(n=2, n_g=64, n_b=2, d=0.5, min_blk=1)
    variants = [
        {}, {"n": 4, "n_b": 2}, {"d": 0.0}, {"d": 1.5}, {"n_g": 400, "d": 0.0025},
        {"n_b": 128}, {"alpha": 1.0}, {"gamma": 1.0}, {"delta0": 0.0},
        {"n_g": 1000, "d": 0.0015}, {"n_g": 1_000_000, "d": 0.001}, {"n_g": 12345, "d": 0.0173},
        {"beta": 1.0}, {"eta": 0.0}, {"blk_move": 0}, {"min_blk": 0}, {"n": 0}, {"n_g": 0},
        {"n_b": 0}, {"max_density_cap": 1.5}, {"max_density_cap": 0.5}, {"n_g": 2_000_001, "d": 0.25},
    ]
    for v in variants:
        kw = dict(base)
        kw.update(v)
        c = O.make_config(**kw)
        o = A.exd_config()
        rc = R.ref_validate(C.byref(c), C.byref(o))
        cases.append({"in": cfg_dict(c), "rc": rc,
                      "k": o.k if rc == 0 else None,
                      "msg": R.ref_last_error().decode() if rc else None})
    out["config"] = cases

    # --- topology (test_partition.cpp:25-95) -------------------------------
    cases = []
    fixed = [(4096, 8, 4, 1), (4096, 5, 2, 1), (64, 2, 2, 1), (64, 4, 2, 1), (4096, 8, 4, 3),
             (4096, 2, 4, 1), (16, 32, 2, 1), (11_200_000, 256, 8, 2), (6_200_000, 256, 8, 2),
             (11_300_000, 256, 8, 2), (11_200_000, 256, 1, 2), (100, 7, 3, 1)]
    for _ in range(300):
        n = int(rng.integers(1, 13))
        mb = int(rng.integers(1, 4))
        nb = n * mb + int(rng.integers(0, 64))
        ng = nb * int(rng.integers(1, 4097))
        fixed.append((ng, nb, n, mb))
    for ng, nb, n, mb in fixed:
        t = A.exd_topology()
        w = C.create_string_buffer(256)
        rc = R.ref_build_topology(ng, nb, n, mb, C.byref(t), w, 256)
        e = {"args": [ng, nb, n, mb], "rc": rc}
        if rc == 0:
            e["topo"] = topo_dict(t)
            e["warning"] = w.value.decode()
            e["ranges"] = []
            for p in range(n):
                st, end = C.c_int64(), C.c_int64()
                R.ref_partition_range(C.byref(t), p, ng, C.byref(st), C.byref(end))
                e["ranges"].append([st.value, end.value])
        else:
            e["msg"] = R.ref_last_error().decode()
        cases.append(e)
    out["topology"] = cases

    # --- allocator (test_allocator.cpp:37-240) -----------------------------
    rot = []
    for kr, t, n in [([5, 9], 1, 2), ([5, 9], 2, 2), ([101, 202, 303], 0, 3)]:
        o = (C.c_int64 * n)()
        R.ref_rotate((C.c_int64 * n)(*kr), t, n, o)
        rot.append({"k_rank": kr, "t": t, "n": n, "out": list(o)})
    for _ in range(200):
        n = int(rng.integers(1, 10))
        t = int(rng.integers(0, 50))
        kr = [int(v) for v in rng.integers(0, 1000, n)]
        o = (C.c_int64 * n)()
        R.ref_rotate((C.c_int64 * n)(*kr), t, n, o)
        rot.append({"k_rank": kr, "t": t, "n": n, "out": list(o)})
    out["rotate"] = rot

    adj = []
    fixed = [(100, [4, 4], [30, 10], 1.25, 1, 1, 800), (100, [4, 4], [20, 20], 1.25, 1, 1, 800),
             (100, [1, 7], [30, 10], 1.25, 1, 1, 800), (100, [4, 4], [10, 30], 1.25, 1, 1, 800)]
    for _ in range(300):
        n = int(rng.integers(2, 10))
        mb = int(rng.integers(1, 3))
        sz = 32 * int(rng.integers(1, 9))
        parts = [mb + int(v) for v in rng.integers(0, 6, n)]
        ng = sum(parts) * sz + int(rng.integers(0, 64))
        k = [int(v) for v in rng.integers(0, 400, n)]
        alpha = float(rng.choice([1.25, 1.1, 1.5, 2.0]))
        fixed.append((sz, parts, k, alpha, int(rng.integers(1, 3)), mb, ng))
    for sz, parts, k, alpha, bm, mb, ng in fixed:
        t = mk_topo(sz, parts)
        kk = (C.c_int64 * len(parts))(*k)
        mv, sk = C.c_int32(), C.c_int32()
        R.ref_adjust(C.byref(t), kk, alpha, bm, mb, ng, C.byref(mv), C.byref(sk))
        adj.append({"sz_blk": sz, "blk_part": parts, "k": k, "alpha": alpha, "blk_move": bm,
                    "min_blk": mb, "n_g": ng, "out_topo": topo_dict(t), "out_k": list(kk),
                    "moves": mv.value, "skips": sk.value})
    out["adjust"] = adj

    alloc = []
    fixed = [(32, [1, 1], 0, 0, 64), (32, [1, 1], 1, 0, 64), (32, [1, 1, 1, 1], 5, 3, 128),
             (30, [1, 1], 0, 1, 70)]
    for _ in range(100):
        n = int(rng.integers(1, 9))
        sz = 16 + int(rng.integers(0, 64))
        parts = [1 + int(v) for v in rng.integers(0, 5, n)]
        ng = sum(parts) * sz + int(rng.integers(0, 32))
        t0 = int(rng.integers(0, 100))
        for r in range(n):
            fixed.append((sz, parts, t0, r, ng))
    for sz, parts, t, r, ng in fixed:
        tp = mk_topo(sz, parts)
        p, st, end = C.c_int32(), C.c_int64(), C.c_int64()
        R.ref_allocate(C.byref(tp), t, r, ng, C.byref(p), C.byref(st), C.byref(end))
        alloc.append({"sz_blk": sz, "blk_part": parts, "t": t, "rank": r, "n_g": ng,
                      "partition": p.value, "range": [st.value, end.value]})
    out["allocate"] = alloc

    # --- threshold (test_threshold.cpp:26-80) ------------------------------
    sc = []
    fixed = [(100, 300, 0.5, 2.0, 0.01), (100, 150, 0.5, 2.0, 0.01), (100, 40, 0.5, 2.0, 0.01),
             (100, 200, 1.0, 2.0, 0.04), (100, 50, 1.0, 2.0, 0.04), (4, 3, 0.5, 2.0, 0.01)]
    for _ in range(500):
        fixed.append((int(rng.integers(1, 1001)), int(rng.integers(0, 5000)),
                      1e-6 + float(rng.random()) * 10.0, 1.001 + float(rng.random()) * 3.0,
                      1e-3 + float(rng.random()) * 0.98))
    for k, kp, d, b, g in fixed:
        sc.append({"k": k, "k_prime": kp, "delta": d, "beta": b, "gamma": g,
                   "out": R.ref_scale_threshold(k, kp, d, b, g)})
    out["scale_threshold"] = sc

    qs = []
    fixed = [([1.0, 2.0, 3.0, 4.0], 0.25), ([4.0, 1.0, 3.0, 2.0], 1.0), ([2.5, 2.5, 2.5], 0.4)]
    for _ in range(50):
        m = int(rng.integers(100, 1000))
        fixed.append(([float(v) for v in np.abs(rng.laplace(size=m))],
                      0.05 + 0.9 * float(rng.random())))
    for mags, d in fixed:
        a = np.array(mags, dtype=np.float64)
        o = C.c_double()
        R.ref_initial_threshold(a.ctypes.data_as(C.POINTER(C.c_double)), len(a), d, C.byref(o))
        qs.append({"mags": mags, "d": d, "out": o.value})
    out["initial_threshold"] = qs

    # --- collectives (test_collectives.cpp:35-119) -------------------------
    gs = []
    lists = [[[1, 4, 9], [2]], [[r * 10 + i for i in range(10)] for r in range(4)],
             [list(range(20))] + [[100 * r + i for i in range(10)] for r in range(1, 4)],
             [[1, 2, 3], [2, 3, 7]], [[], []], [[3, 1]], [[1, 1]]]
    for _ in range(100):
        n = int(rng.integers(2, 8))
        lists.append([[100 * r + i for i in range(int(rng.integers(0, 9)))] for r in range(n)])
    for ls in lists:
        counts = [len(x) for x in ls]
        cat = np.array([v for x in ls for v in x] or [0], dtype=np.int64)
        st = A.exd_gather_stats()
        dups, ul = C.c_int64(), C.c_int64()
        ug = np.zeros(max(1, sum(counts)), dtype=np.int64)
        rc = R.ref_all_gather(cat.ctypes.data_as(O.PI64), (C.c_int64 * len(ls))(*counts), len(ls),
                              C.byref(st), C.byref(dups), ug.ctypes.data_as(O.PI64), C.byref(ul))
        e = {"lists": ls, "rc": rc}
        if rc == 0:
            e.update({"k_prime": st.k_prime, "m_t": st.m_t, "c_t": st.c_t, "f_t": st.f_t,
                      "duplicates": dups.value, "idx_global": [int(v) for v in ug[: ul.value]]})
        else:
            e["msg"] = R.ref_last_error().decode()
        gs.append(e)
    out["gather"] = gs

    # --- the hand-traced engine row (test_engine.cpp:79-131) ---------------
    g0 = [0.6, 0.1, -0.7, 0.2, 0.05, -0.3, 0.9, -0.05]
    g1 = [-0.4, 0.55, 0.1, -0.6, 0.45, 0.2, -0.1, 0.8]
    c = O.make_config(n=2, n_g=8, n_b=2, d=0.5, min_blk=1, delta0=0.5, eta=1.0, beta=2.0,
                      gamma=0.01)
    eng = O.RefEngine(c, O.make_options(parallel_workers=0, verify_conservation=1))
    rec = eng.step([np.array(g0), np.array(g1)], capture=True)
    s0 = eng.state(0)
    out["engine_trace"] = {
        "config": cfg_dict(c), "grads": [g0, g1], "record": A.record_dict(rec),
        "x": [eng.x(r).tolist() for r in range(2)], "e": [eng.e(r).tolist() for r in range(2)],
        "delta": s0.delta, "k_t": list(s0.k_t[:2]), "union": eng.union().tolist(),
    }

    # --- generator (rng.hpp + workloads.cpp) -------------------------------
    gen = []
    for spec_kw in [dict(n_g=4096, seed=7), dict(n_g=5000, seed=99, distribution=1),
                    dict(n_g=3000, seed=5, decay=0.99), dict(n_g=3000, seed=5, decay_step=3),
                    dict(n_g=2000, segments=O.skew_segments(2000), seed=1)]:
        spec = O.stream_spec(**spec_kw)
        for t, r in [(0, 0), (3, 1), (7, 2)]:
            g = O.synthetic_gradient_ref(spec, t, r)
            gen.append({"spec": spec_kw, "t": t, "rank": r,
                        "sha256_f64": hashlib.sha256(g.tobytes()).hexdigest(),
                        "head": g[:16].tolist(), "tail": g[-16:].tolist()})
    out["generator"] = gen

    # --- small multi-step trajectories of the reference Engine -------------
    traj = []
    for kw, segs, iters in [
        (dict(n=3, n_g=6000, n_b=24, d=0.02, seed=11), None, 30),
        (dict(n=4, n_g=9000, n_b=32, d=0.01, seed=3, beta=1.05), "skew", 40),
        (dict(n=2, n_g=4097, n_b=16, d=0.05, seed=5, eta=0.7, delta0=0.8), None, 25),
        (dict(n=1, n_g=3000, n_b=8, d=0.02, seed=9), None, 20),
    ]:
        c = O.make_config(**kw)
        spec_kw = dict(n_g=kw["n_g"], seed=kw["seed"],
                       segments=O.skew_segments(kw["n_g"]) if segs else None)
        spec = O.stream_spec(**spec_kw)
        eng = O.RefEngine(c, O.make_options(verify_conservation=1))
        rows = []
        for t in range(iters):
            gs_ = [O.synthetic_gradient_ref(spec, t, r).astype(np.float32).astype(np.float64)
                   for r in range(c.n)]
            rec = eng.step(gs_, capture=True)
            rows.append({"record": A.record_dict(rec), "union": eng.union().tolist(),
                         "delta_after": eng.state(0).delta,
                         "topo_after": topo_dict(eng.state(0).topology)})
        traj.append({"config": cfg_dict(c), "stream": {k: v for k, v in spec_kw.items()},
                     "grad_rounding": "float32", "rows": rows,
                     "x_sha256": [hashlib.sha256(eng.x(r).tobytes()).hexdigest() for r in range(c.n)],
                     "e_sha256": [hashlib.sha256(eng.e(r).tobytes()).hexdigest() for r in range(c.n)]})
    out["trajectories"] = traj
    # the reference's CSV ledger (runner.cpp:55-80) of the first trajectory
    out["csv"] = {"trajectory": 0, "text": O.ref_format_csv([r["record"] for r in traj[0]["rows"]])}

    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "reference_golden.json"),
          os.path.getsize(os.path.join(HERE, "reference_golden.json")), "bytes")


if __name__ == "__main__":
    main()
