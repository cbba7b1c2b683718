"""Multi-GPU parity check of the one-rank-per-GPU (NCCL) engine.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/dist_check.py [--n_g 200000] [--steps 20]

Every rank runs Engine.rank() on its own GPU with gradients from the device
generator keyed by (t, rank). Rank 0 also regenerates every rank's gradient
on its own GPU (the generator is a pure function of (t, rank), so the bits are
identical), feeds them to the fp32 oracle, and compares the records each step;
at the end every rank's x / e / delta / k_t / topology are gathered (gloo) and
compared with the oracle's replica of that rank. For N <= 2 the NCCL sum is
order-independent, so x must match bit for bit; for N >= 3 x is checked to
1e-6 relative (NCCL's reduction order differs from the reference's rank order).
Exit code 0 on success.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n_g", type=int, default=200_003)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--density", "--d", dest="d", type=float, default=0.01)
    ap.add_argument("--skew", type=int, default=1)
    ap.add_argument("--sync", default="auto", choices=["auto", "nccl", "p2p", "p2p-pull"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--cap", type=float, default=None, help="max_density_cap")
    ap.add_argument("--sparsifier", default="exdyna",
                    choices=["exdyna", "topk", "cltk", "hardthreshold"],
                    help="baseline sparsifiers run over NCCL, checked against oracle.BaselineOracle")
    ap.add_argument("--fixed", type=float, default=2.2, help="hard threshold's fixed_delta")
    ap.add_argument("--kill-peer", type=int, default=0,
                    help="rank 1 stalls after 2 steps; rank 0's next steps must fail with the "
                         "engine's collective error (EXD_ENCCL) instead of hanging")
    ap.add_argument("--inject", type=int, default=0,
                    help="perturb x on rank 1 after step 2; the next step must raise EngineError "
                         "(test_engine.cpp:219-226 across GPUs)")
    ap.add_argument("--mismatch-env", default="",
                    help="KEY=VAL set on rank 1 only before the engine is created; creation must "
                         "fail on every rank with 'differs across ranks' instead of running two "
                         "inbox protocols against each other")
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2402_13781_b200 import sparsim as S

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    kw = dict(n=world, n_g=args.n_g, n_b=max(16, 8 * world), d=args.d, seed=5, beta=1.05,
              max_density_cap=args.cap)
    ids = [S.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    base = args.sparsifier != "exdyna"
    if args.mismatch_env:
        key, val = args.mismatch_env.split("=", 1)
        if rank == 1:
            os.environ[key] = val
        msg = ""
        try:
            S.Engine.rank(S.SparsifierConfig(**kw), S.EngineOptions(dtype=args.dtype, sync=args.sync),
                          rank, local, ids[0]).close()
        except S.InvalidArgument as err:
            msg = str(err)
        good = "differs across ranks" in msg
        flags = [None] * world
        dist.all_gather_object(flags, (good, msg))
        if rank == 0:
            print(f"dist_check world={world} sync={args.sync} mismatch-env {args.mismatch_env}: "
                  f"{'PASS' if all(f[0] for f in flags) else 'FAIL'} {flags}", flush=True)
        dist.destroy_process_group()
        sys.exit(0 if all(f[0] for f in flags) else 1)
    eng = S.Engine.rank(S.SparsifierConfig(**kw),
                        S.EngineOptions(dtype=args.dtype, sync=args.sync, sparsifier=args.sparsifier,
                                        fixed_delta=args.fixed if args.sparsifier == "hardthreshold" else 0.0),
                        rank, local, ids[0])
    segs = O.skew_segments(args.n_g) if args.skew else None
    src = S.SyntheticStream(S.StreamSpec(n_g=args.n_g, segments=segs, seed=5))
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    buf = torch.empty(args.n_g, dtype=tdt, device=f"cuda:{local}")
    ndt = np.float32 if args.dtype == "f32" else np.float64
    if rank != 0:
        orc = None
    elif base:
        orc = O.BaselineOracle(world, args.n_g, S.validate(S.SparsifierConfig(**kw)).k,
                               args.sparsifier, args.fixed if args.sparsifier == "hardthreshold" else 0.0,
                               dtype=ndt)
    else:
        orc = O.OracleEngine(O.make_config(**kw), ndt)
    tmp = torch.empty(args.n_g, dtype=tdt, device=f"cuda:{local}")
    ok = True
    if args.kill_peer:
        import time
        for t in range(2):
            src.gradient(t, rank, buf, args.dtype, eng.stream())
            torch.cuda.synchronize()
            eng.step([buf])
        dist.barrier()
        if rank != 0:
            # a stalled peer: no further collectives from this rank until rank 0
            # has given up (its peer-memory kernels poll for 20 s), then leave
            # without a teardown barrier
            time.sleep(40 if args.sync != "nccl" else 20)
            os._exit(0)
        t0 = time.time()
        msgs = []
        for t in range(2, 4):
            src.gradient(t, rank, buf, args.dtype, eng.stream())
            torch.cuda.synchronize()
            try:
                eng.step([buf])
                msgs.append("no error")
            except S.DeviceError as err:
                msgs.append(str(err))
        el = time.time() - t0
        good = ("did not" in msgs[0] or "asynchronous error" in msgs[0]) and \
            "engine unusable" in msgs[1] and el < 60
        print(f"dist_check world={world} sync={args.sync} ({eng.sync_mode()}) kill-peer: "
              f"{'PASS' if good else 'FAIL'} after {el:.1f} s: {msgs}", flush=True)
        eng.close()
        os._exit(0 if good else 1)
    if args.inject:
        msg = ""
        try:
            for t in range(5):
                src.gradient(t, rank, buf, args.dtype, eng.stream())
                torch.cuda.synchronize()
                eng.step([buf])
                if t == 2 and rank == 1:
                    x = eng.x(0)
                    x[3] += 1.0
                    eng.write(0, "x", x)
        except S.EngineError as err:
            msg = str(err)
        good = msg == "replicated state diverged at iteration 3: rank 1 field x"
        flags = [None] * world
        dist.all_gather_object(flags, (good, msg))
        if rank == 0:
            print(f"dist_check world={world} sync={args.sync} inject: "
                  f"{'PASS' if all(f[0] for f in flags) else 'FAIL'} {flags}", flush=True)
        dist.destroy_process_group()
        sys.exit(0 if all(f[0] for f in flags) else 1)
    for t in range(args.steps):
        src.gradient(t, rank, buf, args.dtype, eng.stream())
        torch.cuda.synchronize()
        rec = eng.step([buf])
        if rank == 0:
            host = []
            for r in range(world):
                src.gradient(t, r, tmp, args.dtype, 0)
                torch.cuda.synchronize()
                host.append(tmp.cpu().numpy().copy())
            orec = orc.step(host)
            o = orec if base else O.A.record_dict(orec)
            for f in ("k_prime", "m_t", "c_t", "f_t", "delta", "density", "eps", "adjust_moves",
                      "adjust_skips", "union_count", "cap_hits", "duplicates", "idle_workers"):
                if getattr(rec, f) != o[f]:
                    print(f"[rank0] t={t} {f}: gpu={getattr(rec, f)} oracle={o[f]}", flush=True)
                    ok = False
            if rec.k_rank != o["k_rank"]:
                print(f"[rank0] t={t} k_rank {rec.k_rank} vs {o['k_rank']}", flush=True)
                ok = False
            if abs(rec.global_err - o["global_err"]) > 1e-6 * max(o["global_err"], 1e-300):
                print(f"[rank0] t={t} global_err {rec.global_err} vs {o['global_err']}", flush=True)
                ok = False
            if not np.array_equal(eng.idx_global().astype(np.int64),
                                  orc.last_union if base else orc.union()):
                print(f"[rank0] t={t} union differs", flush=True)
                ok = False
    st = eng.state(0)
    mine = {"x": eng.x(0), "e": eng.e(0), "delta": st.delta, "k_t": list(st.k_t[:world]),
            "parts": st.topology.parts(), "sel": None if base else eng.selection(0)}
    allst = [None] * world
    dist.all_gather_object(allst, mine)
    if rank == 0:
        for r, m in enumerate(allst):
            if base:
                if m["k_t"] != list(orc.k_t):
                    print(f"[rank0] rank {r} k_t differs", flush=True)
                    ok = False
                oe, ox = orc.e[r], orc.x[r]
            else:
                ost = orc.state(r)
                if m["delta"] != ost.delta or m["k_t"] != list(ost.k_t[:world]) or \
                        m["parts"] != ost.topology.parts():
                    print(f"[rank0] rank {r} control state differs", flush=True)
                    ok = False
                oe, ox = orc.e(r), orc.x(r)
            if not np.array_equal(m["e"], oe):
                print(f"[rank0] rank {r} residual differs ({int(np.sum(m['e'] != oe))})", flush=True)
                ok = False
            if world <= 2 or (args.sync != "nccl" and not base):
                # the peer-memory sync sums in rank order like the reference
                same = np.array_equal(m["x"], ox)
            else:
                # NCCL's reduction order differs from rank order: norm-wise 1e-6
                same = np.max(np.abs(m["x"] - ox)) <= 1e-6 * max(np.max(np.abs(ox)), 1e-30)
            if not same:
                print(f"[rank0] rank {r} x differs (max {np.max(np.abs(m['x'] - ox))})", flush=True)
                ok = False
            if not base and not np.array_equal(m["sel"].astype(np.int64), orc.selection(r)):
                print(f"[rank0] rank {r} selection differs", flush=True)
                ok = False
        print(f"dist_check world={world} sparsifier={args.sparsifier} sync={args.sync} ({eng.sync_mode()}) dtype={args.dtype} cap={args.cap} n_g={args.n_g} steps={args.steps}: "
              f"{'PASS' if ok else 'FAIL'} (last k'={rec.k_prime} f_t={rec.f_t:.3f})", flush=True)
    flag = torch.tensor([1 if ok else 0])
    dist.broadcast(flag, src=0)
    dist.destroy_process_group()
    sys.exit(0 if int(flag[0]) else 1)


if __name__ == "__main__":
    main()
