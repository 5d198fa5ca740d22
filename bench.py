#!/usr/bin/env python
"""Benchmark of the matrix-free DG-CutFEM operator apply (BASELINE.json metric:
"FP64 operator-apply DoFs/s (3D DG CutFEM, k=3) and % roofline vs CSR SpMV").

One step = one cutfem_apply v = A u over the whole C2 workload (BASELINE.json
configs[1]: 64^3 background mesh of [-1,1]^3, sphere r = 0.7, DG Q3, FP64,
u ~ U(-1,1) seeded), inputs resident in HBM.  L2 is flushed (a 2x-L2 write)
before every timed apply; each apply is timed with CUDA events on the launching
stream; max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) the same global workload is split into N x-slabs, one per
GPU, with the NCCL halo exchange inside every apply (strong scaling; DESIGN.md
"Multi-GPU").
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 operator-apply DoFs/s (3D DG CutFEM, k=3)"
UNIT = "DoF/s"

REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


def workload_desc(P, cfg):
    return {"workload": f"{cfg}: DG Q{P.degree} FP64, {P.n_cells[0]}^3 background mesh of "
                        f"[{P.lower[0]:g},{P.lower[0] + P.h * P.n_cells[0]:g}]^3, "
                        + ("sphere r=0.7 at (0.05,0.03,0.02)" if P.level_set.get("type") == "sphere"
                           else "gyroid c=0.3"),
            "degree": P.degree, "n_dofs": P.n_dofs, "n_active": P.n_active, "n_cut": P.n_cut,
            "n_vol_pts": int(P.vol_pts.shape[0]), "n_srf_pts": int(P.srf_pts.shape[0]),
            "n_face_pts": int(P.sf_pts.shape[0]), "l2": "flushed before every timed apply", "host_jitter": "0.1 ms GPU spin queued before each timed step (outside the events)",
            "penalties": "gamma=tau_D=10p^2 (divided by h), GP 0.1 h^(2j-1), j=0..p"}


class ClockSampler:
    """SM clocks / throttle reasons sampled DURING the timed region: in-process NVML
    polling (cheap queries, no process start-up on the box while timing), else an
    `nvidia-smi -lms 100` subprocess."""

    def __init__(self, uuid: str | None):
        self.uuid = uuid
        self.proc = None
        self.lines = []
        self.kind = None
        self._stop = threading.Event()

    def _nvml(self):
        import pynvml
        pynvml.nvmlInit()
        if self.uuid:
            h = pynvml.nvmlDeviceGetHandleByUUID(self.uuid)
        else:
            h = pynvml.nvmlDeviceGetHandleByIndex(0)
        get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

        def poll():
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                    bits = get_reasons(h)
                    self.lines.append(f"{sm}, {mx}, {pw}, {hex(bits)}")
                except Exception:
                    pass
                self._stop.wait(0.02)
        self.th = threading.Thread(target=poll, daemon=True)
        self.th.start()
        self.kind = "nvml"

    def __enter__(self):
        try:
            self._nvml()
            time.sleep(0.05)
            return self
        except Exception:
            pass
        cmd = ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
               "--format=csv,noheader,nounits", "-lms", "100"]
        if self.uuid:
            cmd.insert(1, f"--id={self.uuid}")
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            self.kind = "nvidia-smi"
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.kind == "nvml":
            time.sleep(0.03)
            self._stop.set()
            self.th.join(timeout=1)
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 4:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                bits = int(parts[3], 16)
            except ValueError:
                continue
            sm.append(s)
            mx.append(m)
            for b, name in REASON_BITS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm), "sampler": self.kind}


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic(kernel: str, cfg: str):
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return d.get(cfg, {}).get(kernel)
    except Exception:
        return None


# ----------------------------------------------------------- CPU oracle arm
def oracle_sample(P, target_s: float, seed: int = 0):
    """Time the oracle (as it stands) on a bounded random sample of output blocks."""
    from oracle import Oracle
    O = Oracle(P)
    u = P.seeded_u(0)
    rng = np.random.default_rng(seed)
    order = rng.permutation(P.n_active)
    t0 = time.perf_counter()
    O.apply(u, blocks=order[:8])
    dt = max(time.perf_counter() - t0, 1e-3)
    nb = int(min(P.n_active, max(8, 8 * target_s / dt)))
    blocks = order[:nb]
    t0 = time.perf_counter()
    O.apply(u, blocks=blocks)
    dt = time.perf_counter() - t0
    return nb, dt


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def timed_cores(fn):
    """Run fn(); return (wall seconds, cores actually used = process CPU time / wall)."""
    c0, t0 = time.process_time(), time.perf_counter()
    out = fn()
    dt = time.perf_counter() - t0
    return out, dt, (time.process_time() - c0) / max(dt, 1e-9)


def oracle_csr_rows(P, target_s: float, seed: int = 0):
    """The oracle-assembled CSR rows of a bounded random sample of blocks (cell matrix +
    the face matrices of the block's faces, the oracle's own routines), time-bounded."""
    import scipy.sparse as sp
    from oracle import Oracle
    O = Oracle(P)
    nd = (P.degree + 1) ** 3
    faces_of = {}
    for (m, pl, d, sf) in O.faces:
        faces_of.setdefault(m, []).append((m, pl, d, sf))
        faces_of.setdefault(pl, []).append((m, pl, d, sf))
    order = np.random.default_rng(seed).permutation(P.n_active)
    rows, cols, vals = [], [], []
    loc = np.arange(nd)
    RR, CC = np.meshgrid(loc, loc, indexing="ij")
    t0 = time.perf_counter()
    nb = 0
    for K in order:
        r0 = nb * nd
        blocks = {int(K): O.cell_matrix(int(K))}
        for (m, pl, d, sf) in faces_of.get(int(K), []):
            A = O.face_matrix(m, pl, d, sf)
            own, oth = (0, 1) if m == K else (1, 0)
            for s, b in ((own, int(K)), (oth, pl if m == K else m)):
                blk = A[own * nd:(own + 1) * nd, s * nd:(s + 1) * nd]
                blocks[b] = blocks.get(b, 0) + blk
        for b, blk in blocks.items():
            rows.append((r0 + RR).ravel())
            cols.append((b * nd + CC).ravel())
            vals.append(np.asarray(blk).ravel())
        nb += 1
        if time.perf_counter() - t0 > target_s or nb >= P.n_active:
            break
    M = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(nb * nd, P.n_dofs)).tocsr()
    M.sum_duplicates()
    M.sort_indices()
    return M, nb, time.perf_counter() - t0


def cpu_baseline_line(P, target_s: float):
    """BASELINE.md "CPU-baseline plan": the oracle-assembled CSR SpMV on all host cores
    (plain C + OpenMP, oracle/csrc/spmv.c) and on 1 thread, over the CSR rows of a
    random sample of blocks (a row costs the same in the full matrix), plus the
    oracle's blockwise matrix-forming apply on a sample.  Reported baseline, not the
    optimisation target."""
    from oracle import spmv
    M, nb, t_asm = oracle_csr_rows(P, 0.5 * target_s)
    x = P.seeded_u(0)
    y = np.empty(M.shape[0])
    allc = os.cpu_count() or 1

    def rate(nt):
        spmv.spmv(M, x, y, nthreads=nt)  # warm
        ts = []
        t_end = time.perf_counter() + 1.0
        while len(ts) < 20 or time.perf_counter() < t_end:
            t0 = time.perf_counter()
            spmv.spmv(M, x, y, nthreads=nt)
            ts.append(time.perf_counter() - t0)
            if len(ts) > 2000:
                break
        return M.shape[0] / float(np.median(ts))

    (r_all, _, used_all) = timed_cores(lambda: rate(allc))
    r_one = rate(1)
    (nbf, dtf), _, used_f = timed_cores(lambda: oracle_sample(P, 0.25 * target_s))
    return {"value": r_all, "unit": UNIT, "cores": allc, "kind": "oracle",
            "sample": f"oracle-assembled CSR rows of {nb} random blocks of {P.n_active} "
                      f"({M.shape[0]} rows, {M.nnz} nnz, assembled in {t_asm:.1f} s), C/OpenMP SpMV, "
                      f"median of >= 20 runs / 1 s",
            "what": "oracle CSR SpMV (P:224-227, the paper's sparse baseline P:921-931) on all host cores",
            "cores_busy_measured": round(used_all, 1), "cpu_model": cpu_model(),
            "one_thread": {"value": r_one, "unit": UNIT},
            "forming_apply": {"value": nbf * (P.degree + 1) ** 3 / dtf, "unit": UNIT,
                              "cores_busy_measured": round(used_f, 1),
                              "sample": f"{nbf} random output blocks ({dtf:.1f} s), the oracle's blockwise "
                                        "apply forming every local matrix, numpy fp64"}}


def run_reference(args, P, cfg, rank, world):
    if rank != 0:
        return 0
    n3 = (P.degree + 1) ** 3
    for _ in range(args.warmup):
        oracle_sample(P, 0.5)
    times, nbs = [], []
    c0 = time.process_time()
    for k in range(args.steps):
        nb, dt = oracle_sample(P, args.ref_step_s, seed=k)
        times.append(dt)
        nbs.append(nb)
    dofs = float(np.sum(nbs)) * n3
    value = dofs / float(np.sum(times))
    cores = max(1, int(round((time.process_time() - c0) / max(float(np.sum(times)), 1e-9))))  # busy cores
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_desc(P, cfg),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{int(np.mean(nbs))} random output blocks of {P.n_active} per step "
                                       f"(direct basis evaluation, numpy fp64)",
                             "cores_meaning": "process CPU time / wall time over the timed steps",
                             "host_cores": os.cpu_count(), "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args, P, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2404_07911_b200 as cf
    from paper_2404_07911_b200 import costmodel

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    nd = (P.degree + 1) ** 3
    ug = P.seeded_u(0)
    if world == 1:
        op = cf.CutFEM(P, device=local_rank)
        g0, n_own = 0, P.n_active
        u = torch.from_numpy(ug).to(dev)
        xs = [0, P.n_cells[0]]
    else:
        # x-slab partition (weights 1 / w_cut), one slab per rank, NCCL halo inside the apply
        xs = cf.partition_x(P, world, args.w_cut)
        nid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            nid.copy_(torch.frombuffer(bytearray(cf.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(nid, 0)
        op = cf.CutFEMDist(P, xs[rank], xs[rank + 1], rank, world, bytes(nid.cpu().numpy()), device=local_rank)
        L = cf.LocalProblem(P, xs[rank], xs[rank + 1])
        g0, n_own = L.global_begin, L.n_own
        u = torch.zeros(op.n_ext_dofs, dtype=torch.float64, device=dev)
        u[:n_own * nd] = torch.from_numpy(ug[g0 * nd:(g0 + n_own) * nd]).to(dev)
    st = op.stats()
    v = torch.empty(op.n_dofs, dtype=torch.float64, device=dev)
    props = torch.cuda.get_device_properties(dev)
    l2 = int(getattr(props, "L2_cache_size", 128 << 20) or (128 << 20))
    flush = torch.empty(2 * l2 // 4 + 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def timed(fn, K):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for k in range(K):
            flush.zero_()
            # a short GPU spin before the start event: the host enqueues the whole step
            # while the GPU waits, so host launch jitter stays out of the device timing
            torch.cuda._sleep(200_000)
            evs[k][0].record(stream)
            fn()
            evs[k][1].record(stream)
        torch.cuda.synchronize(dev)
        return np.array([a.elapsed_time(b) for a, b in evs])  # ms

    for _ in range(max(args.warmup, 3)):
        op.apply(u, v)
    torch.cuda.synchronize(dev)

    uuid = None
    try:
        uuid = "GPU-" + str(props.uuid)
    except Exception:
        pass
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(uuid) as clk:
        # the sampler's start-up pause idles the GPU: re-warm (untimed, the same step
        # structure: flush, spin, apply) right before timing
        timed(lambda: op.apply(u, v), 3)
        ms = timed(lambda: op.apply(u, v), args.steps)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms_step = float(ms.mean())
    if world > 1:
        t = torch.tensor([ms_step], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    value = P.n_dofs / (ms_step * 1e-3)  # whole-job throughput: the global operator per step

    # per-kernel timing (attribution) on the same stream
    k_ms = {}
    for which, name in ((0, "structured"), (1, "unstructured")):
        if (which == 0 and st["n_uncut"] == 0) or (which == 1 and st["n_cut"] == 0):
            continue
        for _ in range(2):
            op.apply_kernel(which, u, v)
        k_ms[name] = float(timed(lambda: op.apply_kernel(which, u, v), args.steps).mean())

    own = None
    if world > 1:
        own = np.zeros(P.n_active, bool)
        own[g0:g0 + n_own] = True
    classes = costmodel.face_classes(P, own)
    work = costmodel.apply_work(st, classes)
    peaks = load_peaks()
    bw = float(peaks.get("hbm_gbs", 6543.7)) * 1e9
    fp64 = costmodel.fp64_peak_tflops() * 1e12
    n_ = P.degree + 1
    if n_ <= 3:
        kname = {"structured": f"k_cell<{n_}>", "unstructured": f"k_cut1<{n_}>"}
    elif n_ == 4:
        kname = {"structured": "k_tile2<4,0> + k_uncw<4,8>", "unstructured": "k_cutp<4>"}
    else:
        kname = {"structured": f"k_uncw<{n_}>", "unstructured": f"k_cut<{n_}>"}
    dom = max(k_ms, key=k_ms.get)
    F_dom = work["F_uncut"] if dom == "structured" else work["F_cut"]
    B_dom = work["B_uncut"] if dom == "structured" else work["B_cut"]
    achieved = F_dom / (k_ms[dom] * 1e-3) / 1e12
    traffic = ncu_traffic(kname[dom], cfg)
    t_roof = max(work["F_total"] / fp64, work["B_total"] / bw)
    roofline = {"bound": "alu", "achieved": achieved, "peak": fp64 / 1e12, "unit": "TFLOP/s",
                "frac": achieved / (fp64 / 1e12), "traffic": traffic, "kernel": kname[dom],
                "kernel_ms": k_ms[dom], "flops_per_launch": F_dom, "alg_bytes_per_launch": B_dom,
                "peak_kind": "derived FP64: 148 SM x 64 FMA/clk x 2 x 1.965 GHz",
                "peak_probe": {"value": 34.1, "unit": "TFLOP/s", "what": "DFMA-throughput probe "
                               "(tools/fp64_peak.cu, profiles/r01_fp64_peak.txt); frac vs probe = "
                               + f"{achieved / 34.1:.3f}"},
                "work_model": "SURVEY §8(d) per-unit counts (paper_2404_07911_b200/costmodel.py, pinned by "
                              "tests/test_oracle_pins.py::test_cost_model_*); the dominant kernel's share: "
                              "its cells and the halves of the faces on its side",
                "apply": {"F_alg": work["F_total"], "B_alg": work["B_total"],
                          "flop_per_dof": work["F_total"] / max(op.n_dofs, 1),
                          "byte_per_dof": work["B_total"] / max(op.n_dofs, 1),
                          "t_roof_ms": t_roof * 1e3, "frac": t_roof / (ms_step * 1e-3),
                          "hbm_gbs": bw / 1e9, "fp64_tflops": fp64 / 1e12},
                "per_kernel_ms": k_ms, "scope": "rank 0" if world > 1 else "whole problem",
                "work_counts": {**{k: int(st[k]) for k in ("n_uncut", "n_cut", "n_vol_pts", "n_srf_pts",
                                                               "n_face_pts", "n_dofs", "degree")},
                                **{k: int(v) for k, v in classes.items()}},
                "recompute": "F_cut = n_vol_pts*vol(n) + n_srf_pts*srf(n) + 4*(cutface_side*n^3 + "
                             "cutface_pts_side*(3n^2+4n)) + sipg_side_cut*face(n)/2 + gp_side_cut*gp(n)/2 "
                             "(costmodel.py; DESIGN 5.4); frac = F / kernel_ms / peak"}

    # end to end through the public API with pinned host buffers
    uh = torch.from_numpy(ug[g0 * nd:(g0 + n_own) * nd].copy()).pin_memory()
    vh = torch.empty(op.n_dofs, dtype=torch.float64).pin_memory()
    if world == 1:
        # the steps as one pipelined batch through the public API
        # (cutfem_apply_host_batch): every step copies its u in and its v out, the copy
        # of step k+1's u and of step k-1's v overlapping step k's apply
        uhn = uh.numpy()
        vh2 = torch.empty(op.n_dofs, dtype=torch.float64).pin_memory()
        vhs = [vh.numpy(), vh2.numpy()]
        e2e_batch = lambda K: op.apply_host_batch([uhn] * K, [vhs[k % 2] for k in range(K)])  # noqa: E731
    else:
        def e2e_fn():
            u[:n_own * nd].copy_(uh, non_blocking=True)
            op.apply(u, v)
            vh.copy_(v, non_blocking=True)
            torch.cuda.synchronize(dev)
    if world == 1:
        e2e_batch(2)
        t0 = time.perf_counter()
        e2e_batch(args.steps)
        e2e_s = (time.perf_counter() - t0) / args.steps
        if args.steps % 2 == 0:  # the last step wrote vhs[1]
            vh = vh2
    else:
        for _ in range(2):
            e2e_fn()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_fn()
        e2e_s = (time.perf_counter() - t0) / args.steps
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": P.n_dofs / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * op.n_dofs,
           "d2h_bytes_per_step": 8 * op.n_dofs, "ms_per_step": e2e_s * 1e3,
           "bytes_scope": "per rank" if world > 1 else "whole problem",
           "api": "cutfem_apply_host_batch (pinned host buffers; step k+1's host->device copy and "
                  "step k-1's device->host copy overlap step k's apply)" if world == 1 else
                  "per step: pinned host -> device copy, apply, device -> host copy, sync"}
    vd = op.apply(u, v)
    torch.cuda.synchronize(dev)
    if world == 1:
        assert np.array_equal(vd.cpu().numpy(), vh.numpy()), "host path and device path disagree"

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step,
            "ms_per_step_stats": {"min": float(ms.min()), "median": float(np.median(ms)), "max": float(ms.max()),
                                  "iqr": [float(np.percentile(ms, 25)), float(np.percentile(ms, 75))],
                                  "argmax": int(np.argmax(ms)), "n_above_1.2x_median": int((ms > 1.2 * np.median(ms)).sum())},
            "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {**workload_desc(P, cfg),
                       "parallelism": f"xslab{world}" if world > 1 else "single",
                       "x_split": xs},
            "clocks": clk.summary(), "e2e": e2e,
            "gpu_launches": args.steps * int(st["launches_per_apply"]) * (2 if world > 1 else 1),
            "roofline": roofline}

    if not args.no_csr and world == 1:
        try:
            t0 = time.perf_counter()
            nnz = op.csr_assemble()
            asm_s = time.perf_counter() - t0
            for _ in range(3):
                op.csr_apply(u, v)
            csr_ms = float(timed(lambda: op.csr_apply(u, v), args.steps).mean())
            csr_bytes = 12 * nnz + 16 * P.n_dofs
            line["csr"] = {"value": P.n_dofs / (csr_ms * 1e-3), "unit": UNIT, "ms_per_step": csr_ms,
                           "nnz": nnz, "assemble_s": asm_s, "impl": "cuSPARSE SpMV CSR_ALG1 fp64 int32",
                           "hbm_frac": csr_bytes / (csr_ms * 1e-3) / bw,
                           "speedup_mf_vs_csr": csr_ms / ms_step}
        except Exception as e:  # the comparison path must not hide the main number
            line["csr"] = {"error": str(e)[:200]}

    if args.cg > 0:
        # BASELINE configs[4]: unpreconditioned CG on f = 1 (Dirichlet zero via Nitsche), all in the
        # library's kernels; timed on the device (max over ranks), L2 not flushed between iterations
        b = op.rhs_const(1.0)
        x = torch.zeros(op.n_ext_dofs, dtype=torch.float64, device=dev)
        op.cg(b, x, iters=2)  # warm-up (work vectors)
        x.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        x, hist = op.cg(b, x, iters=args.cg)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        cg_ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([cg_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            cg_ms = float(t.item())
        line["cg"] = {"iters": int(len(hist) - 1), "ms": cg_ms, "ms_per_iter": cg_ms / max(len(hist) - 1, 1),
                      "applies_per_s": (len(hist) - 1) / (cg_ms * 1e-3),
                      "res0": float(hist[0]), "res_final": float(hist[-1]),
                      "apply_share": ms_step * (len(hist) - 1) / cg_ms,
                      "what": "unpreconditioned CG, f = 1, x0 = 0; rhs + dots + axpys in library kernels, "
                              "dots all-reduced over ranks"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_line(P, args.cpu_s)
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--degree", type=int, default=None)
    ap.add_argument("--no-csr", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-s", type=float, default=12.0)
    ap.add_argument("--ref-step-s", type=float, default=3.0)
    ap.add_argument("--w-cut", type=float, default=7.0, help="slab-balance weight of a cut cell (uncut = 1)")
    ap.add_argument("--cg", type=int, default=0, help="also time this many CG iterations (C5: 50)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    import cutgen
    P = cutgen.config(args.config, degree=args.degree)
    if args.impl == "reference":
        return run_reference(args, P, args.config, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    try:
        return run_ours(args, P, args.config, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
