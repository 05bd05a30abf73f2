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
# K4 direct sum, FIO 2D: 2*DFMA + DMUL + DADD per entry = 2*20 + 19 + 15 from
# ncu SASS counters of an 8192 x 65536 sum (profiles/r2_k4.md)
K4_FLOPS_PER_ENTRY = {"fio2d": 74.0}


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
    """DRAM bytes (read + write) per launch of this workload's dominant
    kernel from the committed ncu capture (profiles/r2_traffic.json, else
    r1), or None."""
    for fn in ("r2_traffic.json", "r1_traffic.json"):
        path = os.path.join(ROOT, "profiles", fn)
        try:
            with open(path) as fh:
                rec = json.load(fh).get(config)
        except (OSError, ValueError):
            continue
        if rec and launches == rec.get("launches_per_apply", 1):
            return rec["dram_bytes_per_launch"]
    return None


L2_NOTE = "factor payload > 126 MB L2 except cfg0 / cfg1_unitxi (L2-resident); no flush; vectors L2-resident"


def static_config(name, world):
    """The workload as both arms report it (identical dicts)."""
    if name in ("cfg1", "cfg4", "cfg1_unitxi", "cfg0"):
        n = 64 if name == "cfg0" else 256
        k = 20 if name == "cfg0" else 30
        desc = dict(model="MIDBF 2D FIO", n_per_dim=n, N=n * n, k=k, n0=64, t=5, eps=1e-9,
                    xi="unit grid (Omega = X)" if name == "cfg1_unitxi" else "integer grid [-n/2,n/2)^2")
        nrhs = 64 if name == "cfg4" else 1
    elif name == "cfg2":
        desc = dict(model="MIDBF 2D low-rank phase r=8", n_per_dim=512, N=512 * 512, k=30, n0=64, t=5, eps=1e-9,
                    xi="integer grid", phase="rank-8 rsvd of the explicit 2D FIO phase, q=2, V <- V S")
        nrhs = 1
    elif name == "cfg3":
        desc = dict(model="MIDBF 3D FIO", n_per_dim=32, N=32 ** 3, k=64, n0=64, t=5, eps=1e-9,
                    xi="integer grid [-16,16)^3")
        nrhs = 1
    else:
        raise SystemExit(f"unknown config {name}")
    return dict(workload=name, nrhs=nrhs, parallelism=f"replicas x{world}", l2=L2_NOTE, **desc)


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
                                                    inputs=dict(phase_rank=8, q=2, seconds=t_phase, eps_K=eps_k))
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


def _ref_module():
    """oracle/_ref (the reference's own code, built in the container where
    /root/reference exists; the built files travel to the GPU box), or None."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        import ref as R

        if os.path.exists(R.LIB_PATH):
            R.lib()
            return R
    except Exception:
        pass
    return None


def cpu_baseline(F_path, f, nrhs, budget_s=20.0):
    """The reference's own bf::apply (oracle/_ref: proj/src compiled
    unmodified, Exec::Parallel = OpenMP over groups, src/butterfly.cpp:628)
    on all host cores on the same F, or the oracle restatement when _ref is
    absent: one warm-up, then repeats until the time budget; best and median
    reported, plus one serial apply (the oracle, Exec::Serial)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    R = _ref_module()
    cores = os.cpu_count()
    Fo = O.load(F_path)
    if R is not None:
        Fr = R.Loaded(F_path)
        run, kind, what = (lambda: Fr.apply(f)), "reference", "the reference's bf::apply (oracle/_ref)"
    else:
        run, kind, what = (lambda: Fo.apply(f, parallel=True, threads=cores)), "port", "oracle restatement"
    g = run()
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < 3 or (time.perf_counter() < t_end and len(times) < 200):
        t0 = time.perf_counter()
        g = run()
        times.append(time.perf_counter() - t0)
    t1 = time.perf_counter()
    Fo.apply(f[:, 0] if f.ndim == 2 else f, parallel=False)
    serial = time.perf_counter() - t1
    return g, dict(best=min(times), median=statistics.median(times), reps=len(times), cores=cores,
                   serial_one=serial, kind=kind, what=what)


def accuracy(M, K, F, fk, f):
    """metrics::eps_b (src/metrics.cpp:26-48): rel-L2 of g = F f against the
    direct sum on 256 rows drawn by la::rand_subset(N, 256, mt19937_64(
    chain(0, 0x657062))) (src/experiment.cpp:180), direct sums by K4 on the
    GPU.  For the device-sampled F (K3 entries + K5 IDs, the timed one) and
    a host-sampled F of the same config (entries through the reference's
    EntryFn path on the CPU, host IDs).  SURVEY.md §0: with integer xi no
    k=20/30 factorization is accurate, so both are O(1) and must agree;
    cfg1_unitxi (Omega = X) is the accuracy-meaningful companion."""
    seed = M.chain(0, 0x657062)
    t0 = time.perf_counter()
    e_dev = K.eps_b(F.apply(f), f, nrows=256, seed=seed)
    Fh = M.idbf_factorize(K, fk["n0"], k=fk["k"], eps=1e-9, t=5, seed=M.chain(0, 0x666163), sampler="host",
                          ids="host")
    e_host = K.eps_b(Fh.apply(f), f, nrows=256, seed=seed)
    out = {"eps_b_device_sampled": e_dev, "eps_b_host_sampled": e_host, "rows": 256,
           "rows_seed": "chain(0, 0x657062)", "direct_sum": "K4 on the GPU",
           "host_sampled_total_nnz": Fh.total_nnz, "seconds": time.perf_counter() - t0}
    # K4 throughput on a large direct sum (min(8192, N) rows x N columns)
    nsel = min(8192, F.nrows)
    rows = np.arange(nsel, dtype=np.int64)
    K.direct_sum(f, rows[:256])
    best = 1e9
    for _ in range(3):
        K.direct_sum(f, rows)
        best = min(best, K.last_direct_sum_seconds())
    ent = nsel * F.ncols
    kind = {M.KIND_FIO2D: "fio2d", M.KIND_FIO3D: "fio3d", M.KIND_LOWRANK: "lowrank"}.get(K.desc.kind)
    fpe = K4_FLOPS_PER_ENTRY.get(kind)
    out["k4_direct_sum"] = {"entries": ent, "seconds": best, "entries_per_s": ent / best,
                            "fp64_tflops": ent / best * fpe / 1e12 if fpe else None,
                            "fp64_frac": ent / best * fpe / 1e12 / FP64_DFMA_TFLOPS if fpe else None,
                            "note": "device time (CUDA events) of K4 + its fixed-order reduction, best of 3; "
                                    "ncu: 78.8% FP64 pipe at cfg1 (profiles/r2_k4.md)"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true", help="skip the eps_b key (two direct sums + a host factorize)")
    ap.add_argument("--flags", type=int, default=131135,
                    help="plan flags: 1 PDL | 2 L2 prefetch | 4 graph | 8 persistent dataflow kernel | (v<<4) k1_flow variant (3 = by size) | 512 dense panels | 1024 dense-only k1_flow (default below 200 MB) | 2048 no DMMA | 8192 per-stage DMMA | 65536 never dense-only | 131072 chained single-RHS applies (programmatic dependent launch; default)")
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
    walls, libs = [], []
    for _ in range(3):  # steady state (process-wide pools grown); best of three
        del F
        t0 = time.perf_counter()
        F = M.idbf_factorize(K, fk["n0"], k=fk["k"], eps=1e-9, t=5, seed=M.chain(0, 0x666163), sampler="device")
        walls.append(time.perf_counter() - t0)
        libs.append(F.id_stats()[3])
    t_fac, t_fac_lib = min(walls), min(libs)
    entries, sample_calls, sample_s = F.sample_stats()
    ks = F.kernel_stats()
    k3_rate = ks["k3_entries"] / ks["k3_seconds"] if ks["k3_seconds"] > 0 else None
    fpe = K3_FLOPS_PER_ENTRY.get({M.KIND_FIO2D: "fio2d", M.KIND_FIO3D: "fio3d", M.KIND_LOWRANK: "lowrank"}.get(K.desc.kind))
    k3_line = {"launches": ks["k3_launches"], "entries": ks["k3_entries"], "device_seconds": ks["k3_seconds"],
               "entries_per_s": k3_rate, "k5_launches": ks["k5_launches"], "k5_device_seconds": ks["k5_seconds"],
               "note": "CUDA events around every k3_sample* launch of the timed factorization"}
    if K.desc.kind == M.KIND_FIO2D:  # ncu capture of one cfg1 K3 launch (profiles/r2b_k3.md)
        k3_line["fp64_pipe_busy_ncu"] = {"active": 0.599, "elapsed": 0.564, "source": "profiles/r2b_k3.md"}
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

    apply_ptr, f_ptr, g_ptr = plan.apply_ptr, fd.data_ptr(), gd.data_ptr()

    def step():  # (pointers resolved once: small configs are close to host-issue bound)
        apply_ptr(f_ptr, g_ptr, nrhs, False, sp)

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
            apply_ptr(f_ptr, g_ptr, nrhs, False, sp)
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
    # DRAM bytes actually moved per apply (ncu, cold cache) over the apply time
    frac_dram = (traffic * launches / (ms_step * 1e-3) / 1e9 / hbm) if traffic else None
    if nrhs == 1:
        # algorithmic bytes = the factor as stored (16*total_nnz)
        # + vectors.  k1_flow streams fewer: the ID blocks' exact unit rows /
        # columns are gathered from x (midbf_plan_flow_bytes); the HBM
        # efficiency on the bytes actually streamed is reported beside it.
        streamed = sum(flow_bytes) + vec_bytes
        sgbs = streamed / (ms_step * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "peak_kind": peak_kind, "traffic": traffic, "frac_dram": frac_dram,
                    "algorithmic_bytes_per_apply": alg_bytes,
                    "streamed_bytes_per_apply": streamed, "streamed_gbs": sgbs, "streamed_frac": sgbs / hbm,
                    "note": "achieved = (16*total_nnz + 16*(N_in+N_out)) / apply time (SURVEY.md 8(d): the factor "
                            "as stored); k1_flow streams only the identity-compressed panels (streamed_*), so frac "
                            "can exceed the bandwidth actually used: frac_dram = ncu DRAM bytes (read+write) of the "
                            "launch / apply time / peak is the honest HBM efficiency; "
                            f"one apply = {launches} k1_flow launch in one CUDA graph"}
    else:
        # algorithmic flops = 8 * nrhs * total_nnz; k2_flow skips
        # the exact identity columns of V-type ID strips on 32/64-wide tiles
        flops = 8.0 * F.total_nnz * nrhs
        # real DMMA flops per complex MAC: 32- and 64-wide tiles (slices of
        # 17..64 RHS) use Gauss's three real products (6 flops), 16-wide four
        gauss = not (args.flags & (1 << 26))
        slices = [min(64, nrhs - c) for c in range(0, nrhs, 64)]
        per_mac = sum((6.0 if gauss and w > 16 else 8.0) * w for w in slices) / nrhs
        executed = per_mac * (plan.k2_bytes() / 16) * nrhs
        tf = flops / (ms_step * 1e-3) / 1e12
        etf = executed / (ms_step * 1e-3) / 1e12
        roofline = {"bound": "tensor", "achieved": tf, "peak": FP64_DMMA_TFLOPS, "unit": "TFLOP/s",
                    "frac": tf / FP64_DMMA_TFLOPS, "peak_kind": "measured (tools/fp64_probe.cu, DMMA m8n8k4)",
                    "traffic": traffic, "frac_dram": frac_dram, "algorithmic_flops_per_apply": flops,
                    "executed_flops_per_apply": executed, "executed_tflops": etf,
                    "executed_frac": etf / FP64_DMMA_TFLOPS,
                    "hbm_gbs": achieved, "hbm_frac": achieved / hbm,
                    "dmma_flops_per_complex_mac": per_mac,
                    "note": "achieved = 8*nrhs*total_nnz / apply time (SURVEY.md 8(d)); executed_* = the entries "
                            "k2_flow multiplies (identity columns of V-type strips skipped, midbf_plan_k2_bytes) x the "
                            "real DMMA flops per complex MAC (6 with Gauss's three products on 32- / 64-wide tiles, else 8); "
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
        "config": static_config(args.config, world),
        "inputs": desc.get("inputs"),
        "roofline": roofline,
        "e2e": {"value": replica_throughput(world, nrhs, e_s * 1e3), "unit": "matvecs/s",
                "mode": "pipelined midbf_apply_async over 3 pinned host buffer pairs, CUDA events",
                "sync_value": replica_throughput(world, nrhs, e_sync * 1e3), "result_matches_device": e2e_ok, "h2d_bytes_per_step": 16 * N * nrhs,
                "d2h_bytes_per_step": 16 * F.nrows * nrhs},
        "gpu_launches": launches * args.steps,
        "factorize": {"seconds": t_fac, "library_seconds": t_fac_lib, "wall_seconds_all": walls,
                      "first_call_seconds": t_fac_first, "entries_sampled_on_gpu": entries,
                      "note": "seconds = best wall time of bf::idbf_factorize (KernelDesc overload) over three "
                              "steady-state calls; library_seconds = the factorize proper (trees built, sampler "
                              "uploaded before it)",
                      "sampler_launch_batches": sample_calls, "ids_on_gpu": n_dev_ids, "ids_on_host": n_host_ids,
                      "id_batch_seconds": id_s, "sampler_seconds": sample_s,
                      "total_nnz": F.total_nnz, "factors": F.nfactors, "L": F.L,
                      "k3_sampling": k3_line},
        "stages": [dict(strips=s[0], payload_mb=s[1] / 1e6, flow_mb=b / 1e6, in_len=s[2], out_len=s[3])
                   for s, b in zip(stages, flow_bytes)],
        "clocks": clk.summary(),
        "host_issue_us_per_step": host_issue_us,
    }
    if not args.no_accuracy:
        line["accuracy"] = accuracy(M, K, F, fk, f_host[:, 0])
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        fd_, path = tempfile.mkstemp(suffix=".midbf")
        os.close(fd_)
        F.save(path)
        g_cpu, cb = cpu_baseline(path, f_host if nrhs > 1 else f_host[:, 0], nrhs)
        os.unlink(path)
        g_cpu = g_cpu.reshape((F.nrows, nrhs), order="F")
        err = float(np.linalg.norm(g_dev - g_cpu) / np.linalg.norm(g_cpu))
        line["rel_l2_vs_ref"] = err
        line["rel_l2_vs_ref_note"] = (f"device g vs {cb['what']} on the same F (the product's, handed over as "
                                      "MIDBF001) and f")
        line["cpu_baseline"] = {"value": nrhs / cb["best"], "unit": "matvecs/s", "cores": cb["cores"],
                                "kind": cb["kind"], "median_value": nrhs / cb["median"],
                                "serial_1core_value": 1.0 / cb["serial_one"],
                                "sample": f"{cb['reps']} applies of the same F and f (best of; one warm-up, "
                                          f"~20 s budget): {cb['what']}, OpenMP over groups on all host threads"}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def reference_points(name):
    """Point sets / kernel inputs of a config for the CPU arm (numpy only)."""
    if name in ("cfg1", "cfg4", "cfg1_unitxi", "cfg0"):
        n = 64 if name == "cfg0" else 256
        X = unit_grid(n, 2)
        return X, (X.copy() if name == "cfg1_unitxi" else integer_grid(n, 2)), None, None
    if name == "cfg2":
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import lowrank as LR

        X, Om = unit_grid(512, 2), integer_grid(512, 2)
        allc, allr = np.arange(len(Om)), np.arange(len(X))
        # la::rsvd restated in numpy (oracle/lowrank.py) on the explicit phase,
        # rank 8, q = 2, V <- V S, seed 7: the same recipe as the GPU arm's
        # A, B (equal to rounding; the timing workload is the same shape)
        A, B, _, _ = LR.lowrank_phase(lambda i: LR.fio2d_phase_block(X, Om, [i], allc)[0],
                                      lambda j: LR.fio2d_phase_block(X, Om, allr, [j])[:, 0], len(X), len(Om), 8, 2, 7)
        return X, Om, A, B
    if name == "cfg3":
        return unit_grid(32, 3), integer_grid(32, 3), None, None
    raise SystemExit(f"unknown config {name}")


def reference_arm(args, world, rank):
    """The reference's own CPU path on the same workload: oracle/_ref is
    /root/reference/proj/src compiled unmodified (against the Eigen stand-in
    oracle/shim/, oracle/ref.mk).  Factorize with its bf::idbf_factorize
    (Exec::Parallel, entries from its ker::make_accessor / phase_entry_fn),
    then time its bf::apply with all host threads, each step one apply of
    the experiment's f.  Falls back to the oracle restatement (kind "port")
    only if oracle/_ref is missing.  Under torchrun rank 0 alone runs."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    name = args.config
    cfg = static_config(name, world)
    nrhs, n0, k = cfg["nrhs"], cfg["n0"], cfg["k"]
    X, Om, A, B = reference_points(name)
    kind = {"cfg2": O.KIND_LOWRANK, "cfg3": O.KIND_FIO3D}.get(name, O.KIND_FIO2D)
    R = _ref_module()
    seed = O.chain(0, 0x666163)
    t0 = time.perf_counter()
    if R is not None:
        P = R.Problem(kind, X, Om, A=A, B=B)
        path = P.factorize(n0, k=k, eps=1e-9, t=5, seed=seed, parallel=True)
        Fr = R.Loaded(path)
        apply_fn, total_nnz = Fr.apply, Fr.info["total_nnz"]
        ref_kind, what = "reference", "the reference's bf::idbf_factorize + bf::apply (oracle/_ref, unmodified proj/src)"
    else:
        Ko = O.Kernel(kind, X=X, Omega=Om, A=A, B=B)
        Fo = O.factorize(Ko, X, Om, n0, k=k, eps=1e-9, t=5, seed=seed, parallel=True)
        cores_ = os.cpu_count()
        apply_fn, total_nnz = (lambda f: Fo.apply(f, parallel=True, threads=cores_)), Fo.total_nnz
        ref_kind, what, path = "port", "oracle restatement (oracle/_ref missing)", None
    t_fac = time.perf_counter() - t0
    N = len(Om)
    f = O.random_coefficients(N * nrhs, O.chain(0, 0x66)).reshape((N, nrhs), order="F")
    if nrhs == 1:
        f = f[:, 0]
    cores = os.cpu_count()
    for _ in range(max(1, args.warmup)):
        apply_fn(f)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        g = apply_fn(f)
    s = (time.perf_counter() - t0) / args.steps
    v = nrhs / s
    acc = None
    if R is not None and not args.no_accuracy:
        f1 = f if nrhs == 1 else f[:, 0]
        acc = {"eps_b": P.eps_b(path, f1, 256, O.chain(0, 0x657062)), "rows": 256,
               "rows_seed": "chain(0, 0x657062)", "direct_sum": "metrics::eps_b on the CPU (src/metrics.cpp:26-53)"}
    if path:
        os.unlink(path)
    print(json.dumps({
        "impl": "reference", "metric": "MIDBF matvecs/s at 2D N=256^2 (HBM roofline fraction); rel-L2 err vs ref",
        "value": v, "unit": "matvecs/s", "n_gpus": world, "steps": args.steps, "warmup": max(1, args.warmup),
        "ms_per_step": s * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128 (complex f64)",
        "data": "synthetic (seeded grids + std::mt19937_64 Gaussian f, reference experiment generators)",
        "config": cfg,
        "cpu_baseline": {"value": v, "unit": "matvecs/s", "cores": cores, "kind": ref_kind,
                         "sample": f"{args.steps} applies (after {max(1, args.warmup)} warm-up) of one CPU-built "
                                   f"factorization (total_nnz {total_nnz}): {what}"},
        "e2e": {"value": v, "unit": "matvecs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "factorize_seconds": t_fac,
        "accuracy": acc,
    }))


if __name__ == "__main__":
    main()
