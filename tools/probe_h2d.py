"""Experiment: H2D of one R18 gradient (44.8 MB, pinned) as 1 copy vs chunks on
1-4 streams: does splitting beat one DMA stream on this host's PCIe?"""
import statistics
import torch

n = 11_200_000
h = torch.empty(n, dtype=torch.float32, pin_memory=True).normal_()
d = torch.empty(n, dtype=torch.float32, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
main = torch.cuda.current_stream()


def run(nchunks, nstreams, reps=30):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        step = (n + nchunks - 1) // nchunks
        for i in range(nchunks):
            s = streams[i % nstreams]
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
        for s in streams[:nstreams]:
            main.wait_stream(s)
        e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    return ms, 4 * n / ms / 1e6


for cfg in [(1, 1), (2, 2), (4, 2), (4, 4), (8, 4), (16, 4)]:
    ms, gbs = run(*cfg)
    print(f"chunks={cfg[0]} streams={cfg[1]}: {ms * 1e3:.1f} us, {gbs:.1f} GB/s")
