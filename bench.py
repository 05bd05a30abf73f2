#!/usr/bin/env python
"""MIDBF apply throughput on B200 (BASELINE.json metric).

Workload (default): configs[1] — 2D FIO, n=256 per dim (N=65536), x on the
unit grid, xi on the integer grid [-128,128)^2, k=30, n0=64, t=5, eps=1e-9,
one right-hand side.  The factorization is built by this repo's factorize
with every kernel entry sampled on the GPU (K3) and host IDs; a step is one
MIDBF apply g = F f (K1: 7 stage kernels in one CUDA graph) on a resident f.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
                  [--config cfg0|cfg1|cfg2|cfg3|cfg4|cfg1_unitxi]

One JSON line on rank 0.  Under torchrun each rank builds its own replica
(the apply is not sharded): value = all ranks'
matvecs / max-over-ranks time, scaling "weak".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_SM = 148
# FP64 tensor (DMMA m8n8k4) peak measured on this pool's B200 by tools/fp64_probe.cu
# (MEASURED_PEAKS.json records HBM and bf16 only); DFMA measured 36.7.
FP64_DMMA_TFLOPS = 36.8
FP64_DFMA_TFLOPS = 36.7
# FP64 flops per sampled entry of the K3 samplers (2*DFMA + DMUL + DADD from
# ncu SASS thread counters over whole factorizations divided by the entries
# they sampled; profiles/r1_k3_sample.md), by kernel kind.
K3_FLOPS_PER_ENTRY = {"fio2d": 66.0, "fio3d": 71.0, "lowrank": 60.0}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def integer_grid(n, dim):
    ax = np.arange(-n // 2, n // 2, dtype=np.float64)
    return np.stack(np.meshgrid(*([ax] * dim), indexing="ij"), -1).reshape(-1, dim)


def unit_grid(n, dim):
    ax = np.arange(n, dtype=np.float64) / n
    return np.stack(np.meshgrid(*([ax] * dim), indexing="ij"), -1).reshape(-1, dim)


def measured_traffic(config, launches):
    """DRAM bytes per launch of this workload's dominant kernel from the
    committed ncu capture (profiles/r1_traffic.json), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1_traffic.json")
    try:
        with open(path) as fh:
            rec = json.load(fh).get(config)
    except (OSError, ValueError):
        return None
    if not rec or launches != 1:
        return None
    return rec["dram_bytes_per_launch"]


def workload(name):
    import paper_1908_09376_b200 as M

    if name in ("cfg1", "cfg4", "cfg1_unitxi", "cfg0"):
        n = 64 if name == "cfg0" else 256
        X = unit_grid(n, 2)
        Om = X.copy() if name == "cfg1_unitxi" else integer_grid(n, 2)
        K = M.Kernel(M.KIND_FIO2D, X=X, Omega=Om)
        k = 20 if name == "cfg0" else 30
        desc = dict(model="MIDBF 2D FIO", n_per_dim=n, N=n * n, k=k, n0=64, t=5, eps=1e-9,
                    xi="unit grid (Omega = X)" if name == "cfg1_unitxi" else "integer grid [-n/2,n/2)^2")
        nrhs = 64 if name == "cfg4" else 1
        return K, X, Om, dict(n0=64, k=k), nrhs, desc
    if name == "cfg2":
        n = 512
        X = unit_grid(n, 2)
        Om = integer_grid(n, 2)
        # configs[2]: rank-8 phase factors of the explicit 2D FIO phase from
        # la::rsvd over 16 sampled rows / columns (q = 2), V <- V*Sigma
        # (src/phase_md.cpp:184-224 with recovery = identity), produced by
        # this repo's low-rank phase path (Phi rows / columns on the GPU).
        Kf = M.Kernel(M.KIND_FIO2D, X=X, Omega=Om)
        t0 = time.perf_counter()
        A, B, _, _ = M.lowrank_phase(Kf, 8, 2, seed=7)
        t_phase = time.perf_counter() - t0
        eps_k = M.eps_K(Kf, A, B, 256, 7)
        # point sets define the trees; entries come only from A, B
        K = _lowrank_kernel(M, X, Om, A, B)
        return K, X, Om, dict(n0=64, k=30), 1, dict(model="MIDBF 2D low-rank phase r=8", n_per_dim=n, N=n * n,
                                                    k=30, n0=64, t=5, eps=1e-9, xi="integer grid",
                                                    phase=dict(rank=8, q=2, seconds=t_phase, eps_K=eps_k))
    if name == "cfg3":
        n = 32
        X = unit_grid(n, 3)
        Om = integer_grid(n, 3)
        K = M.Kernel(M.KIND_FIO3D, X=X, Omega=Om)
        return K, X, Om, dict(n0=64, k=64), 1, dict(model="MIDBF 3D FIO", n_per_dim=n, N=n ** 3, k=64, n0=64,
                                                    t=5, eps=1e-9, xi="integer grid [-16,16)^3")
    raise SystemExit(f"unknown config {name}")


def _lowrank_kernel(M, X, Om, A, B):
    K = M.Kernel(M.KIND_LOWRANK, A=A, B=B)
    X = np.ascontiguousarray(X)
    Om = np.ascontiguousarray(Om)
    K._keep += [X, Om]
    K.desc.X, K.desc.Omega, K.desc.dim = M._p(X), M._p(Om), X.shape[1]
    return K


def max_over_ranks(value, world, device):
    """Multi-GPU timing rule: the job time is the slowest rank's time."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_throughput(world, nrhs, ms_per_step):
    """Whole-job matvecs/s: every rank applies its own replica of the
    factorization to nrhs vectors per step (the apply is not sharded,
    DESIGN.md "Multi-GPU"), timed by the slowest rank."""
    return world * nrhs / (ms_per_step * 1e-3)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_baseline(F_path, f, nrhs, budget_s=20.0):
    """Oracle (restated reference apply, OpenMP over groups like
    src/butterfly.cpp:628) on all host cores: one warm-up, then repeats
    until the time budget; best and median reported."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    Fo = O.load(F_path)
    cores = os.cpu_count()
    g = Fo.apply(f, parallel=True, threads=cores)
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < 3 or (time.perf_counter() < t_end and len(times) < 200):
        t0 = time.perf_counter()
        g = Fo.apply(f, parallel=True, threads=cores)
        times.append(time.perf_counter() - t0)
    t1 = time.perf_counter()
    Fo.apply(f[:, 0] if f.ndim == 2 else f, parallel=False)
    serial = time.perf_counter() - t1
    return g, dict(best=min(times), median=statistics.median(times), reps=len(times), cores=cores,
                   serial_one=serial, Fo=Fo)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--flags", type=int, default=63,
                    help="plan flags: 1 PDL | 2 L2 prefetch | 4 graph | 8 persistent dataflow kernel | (v<<4) k1_flow variant (3 = by size) | 512 dense panels | 1024 dense-only k1_flow (default below 200 MB) | 2048 no DMMA | 8192 per-stage DMMA | 65536 never dense-only")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return reference_arm(args, world, rank)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1908_09376_b200 as M

    K, X, Om, fk, nrhs, desc = workload(args.config)
    t0 = time.perf_counter()
    F = M.idbf_factorize(K, fk["n0"], k=fk["k"], eps=1e-9, t=5, seed=M.chain(0, 0x666163), sampler="device")
    t_fac_first = time.perf_counter() - t0  # includes one-time module loading and pool growth
    for _ in range(2):  # the second call still grows process-wide staging pools; time the third
        del F
        t0 = time.perf_counter()
        F = M.idbf_factorize(K, fk["n0"], k=fk["k"], eps=1e-9, t=5, seed=M.chain(0, 0x666163), sampler="device")
        t_fac = time.perf_counter() - t0
    entries, sample_calls, sample_s = F.sample_stats()
    ks = F.kernel_stats()
    k3_rate = ks["k3_entries"] / ks["k3_seconds"] if ks["k3_seconds"] > 0 else None
    fpe = K3_FLOPS_PER_ENTRY.get({M.KIND_FIO2D: "fio2d", M.KIND_FIO3D: "fio3d", M.KIND_LOWRANK: "lowrank"}.get(K.desc.kind))
    k3_line = {"launches": ks["k3_launches"], "entries": ks["k3_entries"], "device_seconds": ks["k3_seconds"],
               "entries_per_s": k3_rate, "k5_launches": ks["k5_launches"], "k5_device_seconds": ks["k5_seconds"],
               "note": "CUDA events around every k3_sample* launch of the timed factorization"}
    if fpe and k3_rate:
        k3_line.update({"fp64_flops_per_entry": fpe, "fp64_tflops": k3_rate * fpe / 1e12, "fp64_peak": FP64_DFMA_TFLOPS,
                        "fp64_frac": k3_rate * fpe / 1e12 / FP64_DFMA_TFLOPS,
                        "peak_kind": "measured DFMA (tools/fp64_probe.cu)"})
    n_dev_ids, n_host_ids, id_s, _ = F.id_stats()
    plan = F.plan(1)
    M.lib().midbf_plan_set_flags(plan._h, args.flags)
    N = F.ncols
    stages = plan.stages()
    flow_bytes = plan.flow_bytes()
    vec_bytes = 16 * nrhs * (F.ncols + F.nrows)
    alg_bytes = 16 * F.total_nnz + vec_bytes  # the factor as stored (every ID block dense)

    f_host = M.random_coefficients(N * nrhs, M.chain(0, 0x66)).reshape((N, nrhs), order="F")
    stream = torch.cuda.current_stream()
    fd = torch.from_numpy(np.asfortranarray(f_host).reshape(-1, order="F").copy()).to("cuda")
    gd = torch.empty(F.nrows * nrhs, dtype=torch.complex128, device="cuda")
    sp = stream.cuda_stream

    def step():
        plan.apply_ptr(fd.data_ptr(), gd.data_ptr(), nrhs, False, sp)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.15)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        h0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        host_issue_us = (time.perf_counter() - h0) / args.steps * 1e6
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # keep the GPU busy a little longer for the clock sampler on short runs
        extra = 0
        t_end = time.perf_counter() + 0.3
        while time.perf_counter() < t_end:
            step()
            extra += 1
        torch.cuda.synchronize()
    ms = max_over_ranks(ev0.elapsed_time(ev1), world, "cuda")
    ms_step = ms / args.steps
    g_dev = gd.cpu().numpy().reshape((F.nrows, nrhs), order="F")

    # e2e through the public API with pinned host operands: every step copies
    # its f host->device and its g device->host.  "e2e" = the pipelined API
    # (midbf_apply_async: copies of step i+1 / i-1 overlap the apply of step
    # i, as a serving loop would run); "e2e_sync" = one blocking call per step.
    host = [(torch.from_numpy(np.asfortranarray(f_host).reshape(-1, order="F").copy()).pin_memory(),
             torch.empty(F.nrows * nrhs, dtype=torch.complex128).pin_memory()) for _ in range(3)]
    fh, gh = host[0]
    for _ in range(3):
        plan.apply_ptr(fh.data_ptr(), gh.data_ptr(), nrhs, False, sp)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = time.perf_counter()
    for _ in range(args.steps):
        plan.apply_ptr(fh.data_ptr(), gh.data_ptr(), nrhs, False, sp)
    torch.cuda.synchronize()
    e_sync = max_over_ranks((time.perf_counter() - e0) / args.steps, world, "cuda")
    for i in range(3):
        plan.apply_async_ptr(host[i][0].data_ptr(), host[i][1].data_ptr(), nrhs, False, sp)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    for i in range(args.steps):
        fh_i, gh_i = host[i % 3]
        plan.apply_async_ptr(fh_i.data_ptr(), gh_i.data_ptr(), nrhs, False, sp)
    eb.record(stream)
    torch.cuda.synchronize()
    e_s = max_over_ranks(ea.elapsed_time(eb) * 1e-3 / args.steps, world, "cuda")
    e2e_ok = all(np.array_equal(h[1].numpy(), gd.cpu().numpy()) for h in host)

    hbm, peak_kind = peaks()
    achieved = alg_bytes / (ms_step * 1e-3) / 1e9
    launches = plan.launches(nrhs)
    traffic = measured_traffic(args.config, launches)
    if nrhs == 1:
        # algorithmic bytes = the factor as stored (16*total_nnz)
        # + vectors.  k1_flow streams fewer: the ID blocks' exact unit rows /
        # columns are gathered from x (midbf_plan_flow_bytes); the HBM
        # efficiency on the bytes actually streamed is reported beside it.
        streamed = sum(flow_bytes) + vec_bytes
        sgbs = streamed / (ms_step * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "peak_kind": peak_kind, "traffic": traffic, "algorithmic_bytes_per_apply": alg_bytes,
                    "streamed_bytes_per_apply": streamed, "streamed_gbs": sgbs, "streamed_frac": sgbs / hbm,
                    "note": "achieved = (16*total_nnz + 16*(N_in+N_out)) / apply time (SURVEY.md 8(d)); k1_flow "
                            "streams only the identity-compressed panels (streamed_*; traffic = ncu DRAM bytes "
                            f"of that launch); one apply = {launches} k1_flow launch in one CUDA graph"}
    else:
        # algorithmic flops = 8 * nrhs * total_nnz; k2_flow skips
        # the exact identity columns of V-type ID strips on 32/64-wide tiles
        flops = 8.0 * F.total_nnz * nrhs
        executed = 8.0 * (plan.k2_bytes() / 16) * nrhs
        tf = flops / (ms_step * 1e-3) / 1e12
        etf = executed / (ms_step * 1e-3) / 1e12
        roofline = {"bound": "tensor", "achieved": tf, "peak": FP64_DMMA_TFLOPS, "unit": "TFLOP/s",
                    "frac": tf / FP64_DMMA_TFLOPS, "peak_kind": "measured (tools/fp64_probe.cu, DMMA m8n8k4)",
                    "traffic": traffic, "algorithmic_flops_per_apply": flops,
                    "executed_flops_per_apply": executed, "executed_tflops": etf,
                    "executed_frac": etf / FP64_DMMA_TFLOPS,
                    "hbm_gbs": achieved, "hbm_frac": achieved / hbm,
                    "note": "achieved = 8*nrhs*total_nnz / apply time (SURVEY.md 8(d)); executed_* = the entries "
                            "k2_flow multiplies (identity columns of V-type strips skipped, midbf_plan_k2_bytes); "
                            f"FP64 tensor-core (DMMA) k2_flow: {launches} cooperative dataflow launch(es) per "
                            "apply (one per 64-RHS slice) in one graph; traffic = DRAM bytes per launch"}
    line = {
        "metric": "MIDBF matvecs/s at 2D N=256^2 (HBM roofline fraction); rel-L2 err vs ref",
        "value": replica_throughput(world, nrhs, ms_step),
        "unit": "matvecs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c128 (complex f64)",
        "data": "synthetic (seeded grids + std::mt19937_64 Gaussian f, reference experiment generators)",
        "config": dict(workload=args.config, nrhs=nrhs, parallelism=f"replicas x{world}",
                       l2="factor payload %.1f MB > 126 MB L2 (no flush needed; vectors L2-resident)"
                          % (16 * F.total_nnz / 1e6), **desc),
        "roofline": roofline,
        "e2e": {"value": replica_throughput(world, nrhs, e_s * 1e3), "unit": "matvecs/s",
                "mode": "pipelined midbf_apply_async over 3 pinned host buffer pairs, CUDA events",
                "sync_value": replica_throughput(world, nrhs, e_sync * 1e3), "result_matches_device": e2e_ok, "h2d_bytes_per_step": 16 * N * nrhs,
                "d2h_bytes_per_step": 16 * F.nrows * nrhs},
        "gpu_launches": launches * args.steps,
        "factorize": {"seconds": t_fac, "first_call_seconds": t_fac_first, "entries_sampled_on_gpu": entries,
                      "sampler_launch_batches": sample_calls, "ids_on_gpu": n_dev_ids, "ids_on_host": n_host_ids,
                      "id_batch_seconds": id_s, "sampler_seconds": sample_s,
                      "total_nnz": F.total_nnz, "factors": F.nfactors, "L": F.L,
                      "k3_sampling": k3_line},
        "stages": [dict(strips=s[0], payload_mb=s[1] / 1e6, flow_mb=b / 1e6, in_len=s[2], out_len=s[3])
                   for s, b in zip(stages, flow_bytes)],
        "clocks": clk.summary(),
        "host_issue_us_per_step": host_issue_us,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        fd_, path = tempfile.mkstemp(suffix=".midbf")
        os.close(fd_)
        F.save(path)
        g_cpu, cb = cpu_baseline(path, f_host if nrhs > 1 else f_host[:, 0], nrhs)
        os.unlink(path)
        g_cpu = g_cpu.reshape((F.nrows, nrhs), order="F")
        err = float(np.linalg.norm(g_dev - g_cpu) / np.linalg.norm(g_cpu))
        line["rel_l2_vs_ref"] = err
        line["cpu_baseline"] = {"value": nrhs / cb["best"], "unit": "matvecs/s", "cores": cb["cores"],
                                "kind": "port", "median_value": nrhs / cb["median"],
                                "serial_1core_value": 1.0 / cb["serial_one"],
                                "sample": f"{cb['reps']} applies of the same F and f (best of; one warm-up), "
                                          "oracle restatement of bf::apply with OpenMP over groups"}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def reference_arm(args, world, rank):
    """The reference's own CPU path (oracle restatement: the reference cannot
    be compiled here) on the same workload: factorize on the CPU, then time
    bf::apply with all host threads."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    name = args.config
    if name not in ("cfg0", "cfg1", "cfg1_unitxi", "cfg4"):
        print(json.dumps({"impl": "reference", "unavailable": f"reference arm wired for 2D FIO configs only ({name})"}))
        return
    n = 64 if name == "cfg0" else 256
    X = unit_grid(n, 2)
    Om = X.copy() if name == "cfg1_unitxi" else integer_grid(n, 2)
    k = 20 if name == "cfg0" else 30
    nrhs = 64 if name == "cfg4" else 1
    K = O.Kernel(O.KIND_FIO2D, X=X, Omega=Om)
    t0 = time.perf_counter()
    Fo = O.factorize(K, X, Om, 64, k=k, eps=1e-9, t=5, seed=O.chain(0, 0x666163), parallel=True)
    t_fac = time.perf_counter() - t0
    f = O.random_coefficients(n * n * nrhs, O.chain(0, 0x66)).reshape((n * n, nrhs), order="F")
    if nrhs == 1:
        f = f[:, 0]
    cores = os.cpu_count()
    for _ in range(max(1, args.warmup)):
        Fo.apply(f, parallel=True, threads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        Fo.apply(f, parallel=True, threads=cores)
    s = (time.perf_counter() - t0) / args.steps
    v = nrhs / s
    print(json.dumps({
        "impl": "reference", "metric": "MIDBF matvecs/s at 2D N=256^2 (HBM roofline fraction); rel-L2 err vs ref",
        "value": v, "unit": "matvecs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": s * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128 (complex f64)", "data": "synthetic",
        "config": {"workload": name, "nrhs": nrhs, "n_per_dim": n, "k": k, "n0": 64},
        "cpu_baseline": {"value": v, "unit": "matvecs/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} applies of one CPU-built factorization (oracle restatement)"},
        "e2e": {"value": v, "unit": "matvecs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "factorize_seconds": t_fac,
    }))


if __name__ == "__main__":
    main()
