"""Experiment: does a CUDA graph of the steady-state step (stream + finish
kernels, PDL edge) shorten the device-timed R18 n=1 step?

    python tools/probe_graph.py [--n_g 11200000] [--steps 200]

Captures two consecutive steps (even / odd parity: the kernels take the step
parity by value) into two graphs and replays them alternately, L2 flushed and
CUDA events around each replay, against the same steps launched on the stream.
Timing only: the host iteration counter runs ahead of the device during capture.
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n_g", type=int, default=11_200_000)
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    import torch
    from cuda.bindings import runtime as rt
    from paper_2402_13781_b200 import sparsim as S
    eng = S.Engine(S.SparsifierConfig(n=1, n_g=a.n_g, n_b=256, d=0.01, seed=7),
                   S.EngineOptions(verify_replication=False))
    src = S.SyntheticStream(S.StreamSpec(n_g=a.n_g, seed=7))
    pool = [torch.empty(a.n_g, device="cuda") for _ in range(2)]
    for i, b in enumerate(pool):
        src.gradient(i, 0, b, "f32", eng.stream())
    torch.cuda.synchronize()
    for i in range(300):
        eng.step_async([pool[i % 2]])
    eng.sync()
    xs = torch.cuda.ExternalStream(eng.stream())
    S.flush_l2(0, eng.stream())

    def timed(launch):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(a.steps)]
        for e0, e1 in evs:
            e0.record(xs)
            e1.record(xs)
        torch.cuda.synchronize()
        for i in range(a.steps):
            S.flush_l2(0, eng.stream())
            evs[i][0].record(xs)
            launch(i)
            evs[i][1].record(xs)
        torch.cuda.synchronize()
        us = [e0.elapsed_time(e1) * 1e3 for e0, e1 in evs]
        return statistics.mean(us), statistics.median(us), min(us)

    stream_res = timed(lambda i: eng.step_async([pool[i % 2]]))
    eng.sync()
    # capture two steps (device t is even here: 300 + steps launched)
    assert eng.iteration() % 2 == 0
    st = rt.cudaStream_t(eng.stream())
    graphs = []
    for k in range(2):
        err, = rt.cudaStreamBeginCapture(st, rt.cudaStreamCaptureMode.cudaStreamCaptureModeRelaxed)
        assert err == rt.cudaError_t.cudaSuccess, err
        eng.step_async([pool[k]])
        err, g = rt.cudaStreamEndCapture(st)
        assert err == rt.cudaError_t.cudaSuccess, err
        err, ge = rt.cudaGraphInstantiate(g, 0)
        assert err == rt.cudaError_t.cudaSuccess, err
        graphs.append(ge)
    graph_res = timed(lambda i: rt.cudaGraphLaunch(graphs[i % 2], st))
    print(f"n_g={a.n_g}: stream launches mean/median/min {stream_res[0]:.2f}/{stream_res[1]:.2f}/"
          f"{stream_res[2]:.2f} us; graph replay {graph_res[0]:.2f}/{graph_res[1]:.2f}/"
          f"{graph_res[2]:.2f} us")


if __name__ == "__main__":
    main()
