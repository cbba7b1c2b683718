"""Multi-GPU step driver for counters (ncu NVLink bytes, nvidia-smi): one rank
per GPU, W warm-up steps and K steps of the push-reduce engine, nothing else.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --no-python \\
        ncu --metrics nvltx__bytes.sum,... -k regex:exchange_kernel ... \\
        python tools/dist_steps.py --n_g 100000000 --density 0.1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n_g", type=int, default=11_200_000)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--sync", default="auto")
    ap.add_argument("--leak", action="store_true",
                    help="exit without the collective teardown (a profiled rank may lag)")
    a = ap.parse_args()
    import time
    import torch
    from paper_2402_13781_b200 import sparsim as S
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    # the NCCL id through a file, not gloo: a rank started under a profiler can
    # take long enough to start that gloo's connect retries run out
    path = f"/tmp/exd_ncclid_{os.environ.get('MASTER_PORT', '0')}"
    if rank == 0:
        nid = S.nccl_unique_id()
        with open(path + ".tmp", "wb") as f:
            f.write(nid)
        os.replace(path + ".tmp", path)
    else:
        t0 = time.time()  # a file left by an earlier run is older than this process
        while not (os.path.exists(path) and os.path.getmtime(path) > t0 - 30):
            time.sleep(0.05)
        nid = open(path, "rb").read()
    cfg = S.SparsifierConfig(n=world, n_g=a.n_g, n_b=256, d=a.density, seed=7)
    eng = S.Engine.rank(cfg, S.EngineOptions(verify_replication=False, sync=a.sync), rank, local,
                        nid)
    src = S.SyntheticStream(S.StreamSpec(n_g=a.n_g, seed=7))
    bufs = [torch.empty(a.n_g, device=f"cuda:{local}") for _ in range(2)]
    for t in range(a.warmup + a.steps):
        src.gradient(t, rank, bufs[t % 2], "f32", eng.stream())
        eng.step_async([bufs[t % 2]])
        if t % 8 == 7:
            rec = eng.sync()
    rec = eng.sync()
    if rank == 0:
        print(f"dist_steps world={world} n_g={a.n_g} d={a.density} sync={eng.sync_mode()} "
              f"t={rec.t} k'={rec.k_prime} k_rank={rec.k_rank}", flush=True)
    if rank == 0 and os.path.exists(path):
        os.remove(path)
    if a.leak:
        eng.h = None  # the driver reclaims everything at exit
        return
    eng.close()  # the teardown barrier is collective (NCCL)


if __name__ == "__main__":
    main()
