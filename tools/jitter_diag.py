import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, cutgen, paper_2404_07911_b200 as cf
P = cutgen.config("C2"); op = cf.CutFEM(P)
u = torch.from_numpy(P.seeded_u(0)).cuda(); v = torch.empty_like(u)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
for spin in (200_000, 2_000_000):
    for rep in range(2):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(40)]
        for a, b in evs:
            flush.zero_(); torch.cuda._sleep(spin); a.record(st); op.apply(u, v); b.record(st)
        torch.cuda.synchronize()
        ms = np.array([a.elapsed_time(b) for a, b in evs])
        print(spin, rep, "mean %.4f median %.4f max %.4f n>1.2med %d argmax %d" % (ms.mean(), np.median(ms), ms.max(), (ms > 1.2*np.median(ms)).sum(), ms.argmax()))
