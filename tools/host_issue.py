"""Host issue cost of back-to-back device applies (MIDBF_HOST_TIMING=1 prints
the per-phase breakdown): python tools/host_issue.py [config] [n]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1908_09376_b200 as M

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg0"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
K, X, Om, fk, nrhs, desc = bench.workload(cfg)
F = M.idbf_factorize(K, fk["n0"], k=fk["k"], eps=1e-9, seed=M.chain(0, 0x666163))
plan = F.plan(1)
f = torch.randn(F.ncols, dtype=torch.complex128, device="cuda")
g = torch.empty(F.nrows, dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(50):
    plan.apply_ptr(f.data_ptr(), g.data_ptr(), 1, False, s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(n):
    plan.apply_ptr(f.data_ptr(), g.data_ptr(), 1, False, s)
t_issue = time.perf_counter() - t0
e1.record()
torch.cuda.synchronize()
print(f"{cfg}: host issue {t_issue / n * 1e6:.2f} us/apply, device {e0.elapsed_time(e1) / n * 1e3:.2f} us/apply")
