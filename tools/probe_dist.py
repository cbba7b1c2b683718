"""Experiment: per-step timeline of the one-rank-per-GPU step (torchrun).
EXD_LIB=paper_2402_13781_b200/lib/libexdyna_probe.so torchrun --nproc-per-node 2 tools/probe_dist.py --sync p2p
"""
import argparse, ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser(); ap.add_argument("--sync", default="p2p")  # p2p | p2p-pull | nccl
ap.add_argument("--flush", type=int, default=0)
ap.add_argument("--n_g", type=int, default=11_200_000)
ap.add_argument("--density", type=float, default=0.01)
ap.add_argument("--warm", type=int, default=300)
a = ap.parse_args()
import torch, torch.distributed as dist
from paper_2402_13781_b200 import sparsim as S
from paper_2402_13781_b200._lib import lib
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank)); torch.cuda.set_device(local)
dist.init_process_group("gloo")
ids = [S.nccl_unique_id() if rank == 0 else None]; dist.broadcast_object_list(ids, src=0)
n_g = a.n_g
eng = S.Engine.rank(S.SparsifierConfig(n=world, n_g=n_g, n_b=256, d=a.density, seed=7),
                    S.EngineOptions(sync=a.sync, verify_replication=False), rank, local, ids[0])
src = S.SyntheticStream(S.StreamSpec(n_g=n_g, seed=7))
bufs = [torch.empty(n_g, device=f"cuda:{local}") for _ in range(2)]
for i, b in enumerate(bufs): src.gradient(i, rank, b, "f32", eng.stream())
torch.cuda.synchronize()
for i in range(a.warm): eng.step_async([bufs[i % 2]])
eng.sync(); dist.barrier()
xs = torch.cuda.ExternalStream(eng.stream())
NS = 50 if n_g < 50_000_000 else 10
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(NS)]
for i in range(NS):
    if a.flush: S.flush_l2(local, eng.stream())
    evs[i][0].record(xs); eng.step_async([bufs[i % 2]]); evs[i][1].record(xs)
eng.sync()
us = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in evs)
out = f"rank {rank} sync={eng.sync_mode()} n_g={n_g} d={a.density} flush={a.flush}: step median {us[len(us) // 2]:.1f} us min {us[0]:.1f} max {us[-1]:.1f}"
L = lib()
if hasattr(L, "exd_debug_probe"):
    L.exd_debug_probe.argtypes = [C.POINTER(C.c_uint64)]
    buf = (C.c_uint64 * 64)(); L.exd_debug_probe(buf)
    t0 = buf[16]
    if eng.sync_mode() == "p2p":  # push-reduce exchange kernel
        names = {16: "k1", 17: "k1_last", 0: "x_start", 1: "h1_sent", 2: "h1_in", 8: "w0_gate0",
                 41: "max_base", 42: "max_stage_ld", 43: "max_put", 45: "max_pass1", 9: "w0_done", 44: "max_done",
                 4: "epi_end"}
        out += f"  | prev step: k1 -> max_done {(buf[50]-buf[51])/1e3:.1f} us, max_done -> this k1 {(buf[16]-buf[50])/1e3:.1f} us"
    else:
        names = {16: "k1", 17: "k1_last", 8: "k2copy0", 0: "k2epi", 3: "k2epi_end", 20: "sync", 21: "counts_in", 22: "contrib_done", 23: "contribs_in", 24: "epi_end", 25: "b0_end"}
    out += "  | " + "  ".join(f"{v}={(buf[k]-t0)/1e3:.1f}" for k, v in sorted(names.items(), key=lambda kv: buf[kv[0]]) if buf[k])
print(out, flush=True)
dist.barrier(); dist.destroy_process_group()
