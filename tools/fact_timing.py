import sys, os, time
sys.path.insert(0, os.getcwd())
import bench, paper_1908_09376_b200 as M
for cfgname in sys.argv[1:]:
    K, X, Om, fk, nrhs, desc = bench.workload(cfgname)
    for rep in range(3):
        t=time.perf_counter(); F = M.idbf_factorize(K, fk["n0"], k=fk["k"], eps=1e-9, t=5, seed=M.chain(0, 0x666163)); dt=time.perf_counter()-t
        print(cfgname, rep, f"{dt*1e3:.1f} ms", F.id_stats(), F.kernel_stats(), file=sys.stderr, flush=True)
        del F
