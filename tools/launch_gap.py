import torch, sys, os
sys.path.insert(0, "/root/repo")
from paper_2402_13781_b200 import sparsim as S
torch.cuda.init()
s = torch.cuda.current_stream()
t = torch.zeros(16, device="cuda")
big = torch.zeros(11_200_000, device="cuda")
def run(label, fn, flush=True):
    vals = []
    for i in range(20):
        if flush:
            S.flush_l2(0, s.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); fn(); e1.record(s)
        torch.cuda.synchronize()
        vals.append(e0.elapsed_time(e1) * 1e3)
    vals.sort()
    print(f"{label}: median {vals[10]:.1f} us min {vals[0]:.1f}")
run("nothing", lambda: None)
run("tiny kernel", lambda: t.add_(1))
run("two tiny kernels", lambda: (t.add_(1), t.add_(1)))
run("11.2M add_", lambda: big.add_(1))
run("11.2M add_ noflush", lambda: big.add_(1), flush=False)
