#!/usr/bin/env python
"""TT-UTV throughput benchmark (BASELINE.json metric: tensor entries/s, FP64).

Default workload (N=1): BASELINE config 3 -- the largest single-GPU config: a 24^6
tensor (191M entries, 1.53 GB) from random N(0,1) TT cores of ranks 20 plus 1e-4 relative
Gaussian noise, built with the reference's own generator algorithms (inputs.py, bitwise
the reference's buffers). One step = one TT-ULV left-to-right plus one TT-URV right-to-left
decomposition at fixed rank 20 of the whole tensor (2 x 191M entries).
Default at N > 1 (torchrun, or spawned by this script): config 5 (1024^3, fixed rank 128,
TT-URV) column-sharded across the ranks (one tensor, strong scaling).

  value   entries/s with the tensor resident in HBM (device-timed, CUDA events on the
          engine's stream, max over ranks)
  e2e     the same through the public API from pinned host memory: H2D of the tensor
          and D2H of every core inside the timed region; the step's two independent
          decompositions are issued from two host threads (the API is reentrant, each
          thread has its own stream), so one's H2D overlaps the other's compute
          (--e2e-concurrency 1: back to back; the JSON carries both)
  roofline  the dominant kernel (pass-1 streaming GEMV, HBM-bound) timed live with
          CUDA events around each launch inside the timed region, plus the whole-step
          T_roof / T_dev of SURVEY.md 8(d) (F_min / P_FP64 vs B_comp / BW per cut, P_FP64
          a cuBLAS DGEMM measured in this run -- measurement only, never the product path)
  cpu_baseline  the reference CPU library (oracle/_ref, compiled from /root/reference)
          on this host's cores, on a bounded sample, rank 0 only

`--impl reference` times the reference CPU implementation itself on the whole workload
(the full tensor, both decompositions per step).
`--config {1,2,3,5}` selects another BASELINE config (parity/extra measurements).
Multi-GPU: configs 1-3 do not shard, so every rank runs an independent replica
("replicas only", scaling weak); config 5 runs the column-sharded TT-URV.
"""
from __future__ import annotations

import argparse
import threading
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))

METRIC = "TT-UTV tensor entries/sec (FP64)"
UNIT = "entries/s"
FALLBACK_HBM = 6650.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def workload(cfg: int):
    from paper_2501_07904_b200.inputs import CONFIGS
    c = CONFIGS[cfg]
    runs = [("ulv", "l2r"), ("urv", "r2l")]
    desc = {1: "cfg1 20^4 planted TT (1,5,5,5,1) + 1e-8 noise, fixed rank",
            2: "cfg2 Hilbert-type 32^5 A=1/(i1+..+i5-4), rank-adaptive eps=1e-8",
            3: "cfg3 24^6 planted TT ranks 20 + 1e-4 noise, fixed rank 20",
            5: "cfg5 1024^3 planted TT (1,128,128,1) + 1e-6 noise, fixed rank 128"}[cfg]
    if cfg == 5:
        runs = [("urv", "r2l")]
    return c, runs, desc


def host_cpu():
    """Model name, logical threads and physical cores of this host (cpu_baseline.cores is
    the thread count actually used)."""
    model, phys = None, set()
    try:
        cur = {}
        for line in open("/proc/cpuinfo"):
            if ":" not in line:
                if "physical id" in cur and "core id" in cur:
                    phys.add((cur["physical id"], cur["core id"]))
                cur = {}
                continue
            k, v = (x.strip() for x in line.split(":", 1))
            cur[k] = v
            if k == "model name" and model is None:
                model = v
        if "physical id" in cur and "core id" in cur:
            phys.add((cur["physical id"], cur["core id"]))
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count(), "physical_cores": len(phys) or None}


def measure_fp64_peak(device):
    """Dense FP64 peak of this GPU: cuBLAS DGEMM (torch.matmul, float64) on 8192^3, best of 5
    after warm-up. Measurement only (the roofline's P_FP64); the engine
    never calls cuBLAS."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=device)
    b = torch.randn(n, n, dtype=torch.float64, device=device)
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = None
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    del a, b
    torch.cuda.empty_cache()
    return {"tflops": 2.0 * n ** 3 / (best * 1e-3) / 1e12, "how": f"cuBLAS DGEMM {n}^3 (torch.matmul float64), "
            "best of 5 with CUDA events, measured in this run"}


def golden_parity(cfg: int, a_host, info: dict):
    """The reference's own results on this exact input (tests/golden/full_cfg{cfg}.npz,
    produced by the reference on its own generators; the input is bitwise the same -- its
    norm and sum are checked) beside ours."""
    path = ROOT / "tests" / "golden" / f"full_cfg{cfg}.npz"
    if not path.exists():
        return None
    import numpy as np
    g = np.load(path)
    # config 2 is deterministic (no seed); its golden holds the neutral-rescaling study, scale 1 first
    pre = "e8_s0_" if cfg == 2 else ""
    same = (a_host is not None and (cfg == 2 or
            abs(float(a_host.sum()) - float(g["a_sum"])) <= 1e-9 * abs(float(g["a_sum"])) + 1e-300))
    out = {"input_matches_golden": bool(same), "source": f"tests/golden/full_cfg{cfg}.npz (reference, oracle/_ref)"}
    for m, r in info.items():
        if f"{pre}{m}_ranks" not in g:
            continue
        ref_rse = float(g[f"{pre}{m}_rse"]) if f"{pre}{m}_rse" in g else None
        out[m] = {"ranks_ours": r["ranks"], "ranks_reference": [int(x) for x in g[f"{pre}{m}_ranks"]],
                  "rse_ours": r.get("rse"), "rse_reference": ref_rse,
                  "abs_rse_diff": (abs(r["rse"] - ref_rse) if (ref_rse is not None and r.get("rse") is not None)
                                   else None)}
    return out


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        if os.environ.get("BENCH_NO_SMI") == "1":  # diagnostics: no sampler
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "250"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self, t_begin=None, t_end=None, windows=None):
        """Stops the sampler; summary of the samples inside [t_begin, t_end] (and of each extra
        (t0, t1) in `windows`, returned as a list after it)."""
        if not self.proc:
            return None if windows is None else (None, [None] * len(windows))
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        self.proc = None
        all_rows = [r.split(",") for r in out.strip().splitlines() if r.count(",") >= 8]
        if windows is None:
            return self._summary(all_rows, t_begin, t_end)
        return self._summary(all_rows, t_begin, t_end), [self._summary(all_rows, a, b) for a, b in windows]

    def _summary(self, all_rows, t_begin, t_end):
        rows = list(all_rows)
        if t_begin is not None:
            import datetime
            inside = []
            for r in rows:
                try:
                    ts = datetime.datetime.strptime(r[0].strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    continue
                if t_begin - 0.15 <= ts <= t_end + 0.15:
                    inside.append(r)
            rows = inside or rows[-2:]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for name, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(rows)}


def dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        import torch
        torch.cuda.set_device(local)
        dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = dist_mod
    return world, rank, local, dist


def max_over_ranks(x: float, dist) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def ncu_traffic(cfg: int, kernel: str = ""):
    """ncu DRAM traffic of one launch of `kernel` on this config (profiles/traffic.json:
    entries keyed by config, optionally with a suffix, each naming its kernel)."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        d = json.loads(p.read_text())
    except Exception:
        return None
    t = None
    for key, v in d.items():
        if (key == str(cfg) or key.startswith(f"{cfg}_")) and v.get("kernel") and kernel.startswith(v["kernel"]):
            t = v
            break
    if t is None:
        t = d.get(str(cfg))
        if t is not None and t.get("kernel") and kernel and not kernel.startswith(t["kernel"]):
            t = None  # that capture is of another kernel
    # the DRAM peak ncu implies is a property of the part, not of the config
    if t is not None and "implied_dram_peak_gbs_ncu" not in t:
        for v in d.values():
            if "implied_dram_peak_gbs_ncu" in v:
                t = dict(t, implied_dram_peak_gbs_ncu=v["implied_dram_peak_gbs_ncu"])
                break
    return t


def reference_step(ref, a_host, c, runs, keep=False):
    """One step of the reference CPU library on the host buffer (its stock decompose())."""
    out = []
    for method, sweep in runs:
        if c["mode"] == "tol":
            rr = ref.decompose(a_host, c["dims"], method, sweep, eps=c["eps"])
        else:
            rr = ref.decompose(a_host, c["dims"], method, sweep, ranks=c["ranks"])
        out.append(rr if keep else rr.ranks_chosen)
    return out


def run_reference(args):
    world, rank, local, dist = dist_setup(args.gpus)
    c, runs, desc = workload(args.config)
    if rank != 0:
        return 0
    from oracle import ref
    from paper_2501_07904_b200.inputs import build_host
    a = build_host(args.config)  # the same buffer as our arm (bitwise the reference's generators)
    dims = c["dims"]
    cs = dict(c)
    n = a.size
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    small = ref.gen_gaussian([8, 8, 8], 1)
    # Warm-up: the OpenMP pool on a tiny problem (the first parallel region costs ~1 s); a
    # full-size untimed step would only repeat the timed work at minutes per step.
    for _ in range(args.warmup):
        ref.decompose(small, [8, 8, 8], "urv", "r2l", ranks=[1, 3, 3, 1])
    t0 = time.perf_counter()
    got = None
    per_step = []
    # Every timed step is the whole workload (no slicing). The CPU needs ~90 s per config-3
    # step on 16 threads, so the loop stops once --ref-budget-s of timed work is done (at
    # least one step) and reports the steps it actually timed.
    for i in range(args.steps):
        ts = time.perf_counter()
        got = reference_step(ref, a, cs, runs, keep=True)
        per_step.append(time.perf_counter() - ts)
        log(f"reference step {i}: {per_step[-1]:.1f} s")
        if time.perf_counter() - t0 >= args.ref_budget_s:
            break
    dt = time.perf_counter() - t0
    timed = len(per_step)
    value = timed * len(runs) * n / dt
    ranks = [r.ranks_chosen for r in got]
    rses = []
    for r in got:  # outside the timed region
        try:
            rses.append(ref.rse(r, a, dims, cap=2 * 10**9) if n <= 4 * 10**8 else None)
        except Exception:
            rses.append(None)
    note = "the whole tensor"
    sample = (f"{timed} timed step(s) of {desc} ({len(runs)} decomposition(s) each) on {note}, dims {dims}, "
              f"ranks {ranks}, rse {rses}, seconds per step {[round(x, 2) for x in per_step]}"
              + (f"; stopped after {timed} of the {args.steps} requested steps at the {args.ref_budget_s:.0f} s "
                 "timed-work budget" if timed < args.steps else ""))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": timed,
            "steps_requested": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / timed, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "entries_per_step": len(runs) * n, "parallelism": "cpu-openmp",
                       "ranks": {m: r for (m, _), r in zip(runs, ranks)},
                       "rse": {m: x for (m, _), x in zip(runs, rses)}},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample,
                             "cpu": host_cpu()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    world, rank, local, dist = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    from paper_2501_07904_b200 import api
    from paper_2501_07904_b200._native import lib, check
    from paper_2501_07904_b200.inputs import build_host
    from paper_2501_07904_b200.roofline import step_roofline
    check(lib().ttg_set_device(local))
    c, runs, desc = workload(args.config)
    a_host = build_host(args.config)  # bitwise the reference generators' buffer (inputs.py)
    a = torch.from_numpy(a_host).to(torch.device("cuda", local))
    if world > 1 or args.config == 5:
        pass  # config 5's 8.6 GB host copy is kept for the CPU baseline sample only
    torch.cuda.synchronize()
    fp64 = measure_fp64_peak(torch.device("cuda", local)) if rank == 0 else None
    n = a.numel()
    dims = c["dims"]
    stream = torch.cuda.ExternalStream(lib().ttg_stream(), device=torch.device("cuda", local))
    sharded = args.sharded or (args.config == 5 and world > 1)

    def kw(method):
        return dict(eps=c["eps"]) if c["mode"] == "tol" else dict(ranks=c["ranks"])

    comm = None
    blk = None
    if sharded:
        # one NCCL communicator for the engine; its unique id travels over torch.distributed
        obj = [api.nccl_unique_id() if rank == 0 else None]
        if dist:
            dist.broadcast_object_list(obj, src=0)
        comm = api.nccl_comm(obj[0], world, rank)
        method = runs[0][0]
        lo, hi, rows, cols = api.shard_range(dims, method, world, rank)
        if method == "ulv":
            blk = a[rows * lo:rows * hi].clone()
        else:  # rows [lo, hi) of c = A(i1..i(d-1); id): an (hi-lo) x Id column-major block
            blk = a.view(cols, n // cols)[:, lo:hi].contiguous()
        del a
        torch.cuda.empty_cache()
        a = None
    src = blk if sharded else a

    info = {}

    def step_device():
        for method, sweep in runs:
            if sharded:
                res = api.decompose_sharded(blk.data_ptr(), dims, comm, method, sweep, a_is_device_ptr=True,
                                            qlp=args.qlp, **kw(method))
            else:
                res = api.decompose_device(a.data_ptr(), dims, method, sweep, a_is_device_ptr=True, qlp=args.qlp,
                                           **kw(method))
            info[method] = res
        return info

    # The nvidia-smi sampler starts before the warm-up so its start-up (fork + NVML init)
    # never overlaps the timed region; only samples inside the region are kept.
    clocks = Clocks(local)
    clocks.start()
    # Kernel event timing is on during the warm-up too, so the timed region reuses the
    # pooled CUDA events instead of creating them.
    lib().ttg_profile_enable(1)
    for _ in range(args.warmup):
        step_device()
    # ---- timed region: tensor resident in HBM ----
    d0, d1 = C_double(), C_double()
    lib().ttg_profile_read(ctypes.byref(d0), ctypes.byref(d1))  # discard warm-up records
    lib().ttg_profile_reset_kernels()
    big_ph = (ctypes.c_double * 24)()
    lib().ttg_profile_big_phases(big_ph, 1)  # zero the persistent loop's phase totals
    launches0 = lib().ttg_kernel_launches()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t_begin = time.time()
    e0.record(stream)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    for i in range(args.steps):
        ts = time.perf_counter()
        marks[i].record(stream)
        step_device()
        log(f"step {i}: {1e3 * (time.perf_counter() - ts):.1f} ms host wall")
    marks[-1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    t_end = time.time()
    if dist:
        dist.barrier()
    launches = lib().ttg_kernel_launches() - launches0
    ms = e0.elapsed_time(e1)
    log("device ms per step: " + " ".join(f"{marks[i].elapsed_time(marks[i + 1]):.1f}" for i in range(args.steps)))
    nk = lib().ttg_profile_read(ctypes.byref(d0), ctypes.byref(d1))
    lib().ttg_profile_enable(0)
    lib().ttg_profile_big_phases(big_ph, 0)  # the timed steps' persistent-loop phase totals
    kern_ms, kern_bytes = d0.value, d1.value
    ms_max = max_over_ranks(ms, dist)
    entries_per_step = len(runs) * n
    jobs = 1 if sharded else world  # sharded: one tensor across the ranks (strong scaling)
    value = jobs * args.steps * entries_per_step / (ms_max * 1e-3)

    rep = {m: r.report() for m, r in info.items()}
    rse = {m: r.rse(a.data_ptr(), on_device=True) for m, r in info.items()} if not sharded else {}
    info.clear()
    seq_ms_max = ms_max

    clk = clocks.stop(t_begin, t_end)

    # ---- e2e: public API from pinned host memory, H2D + D2H inside the timed region ----
    host = torch.empty(src.numel(), dtype=torch.float64, pin_memory=True)
    host.copy_(src.reshape(-1))
    torch.cuda.synchronize()
    def e2e_one(method, sweep):
        # one decomposition through the public API: H2D of the tensor inside the call, D2H
        # of every core; returns the bytes moved
        if sharded:
            res = api.decompose_sharded(host.data_ptr(), dims, comm, method, sweep, qlp=args.qlp, **kw(method))
        else:
            res = api.decompose_device(host.data_ptr(), dims, method, sweep, qlp=args.qlp, **kw(method))
        return src.numel() * 8, sum(res.core(k).nbytes for k in range(res.order()))

    def e2e_run(concurrent):
        # concurrent: the step's independent decompositions (ULV, URV) are issued from one
        # host thread each -- the API is reentrant: uploads run one at a time at the full
        # host-link rate and decompositions take the device in turn, so the second tensor's
        # H2D overlaps the first decomposition's compute. The threads are joined at the end of
        # every step (letting them run on through the steps measured anywhere between 3.4e9
        # and 6.1e9 entries/s on the B200; joined per step it is stable).
        moved = []
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            if concurrent:
                out = [None] * len(runs)
                errs = []

                def work(i, m, s):
                    try:
                        # a new host thread starts on device 0: select this rank's GPU first
                        torch.cuda.set_device(local)
                        check(lib().ttg_set_device(local))
                        out[i] = e2e_one(m, s)
                    except Exception as e:  # reported after the join
                        errs.append(e)

                th = [threading.Thread(target=work, args=(i, m, s)) for i, (m, s) in enumerate(runs)]
                for x in th:
                    x.start()
                for x in th:
                    x.join()
                if errs:
                    raise errs[0]
                moved += out
            else:
                moved += [e2e_one(m, s) for m, s in runs]
        secs = max_over_ranks(time.perf_counter() - t0, dist)
        return secs, sum(a for a, _ in moved), sum(b for _, b in moved)

    conc = args.e2e_concurrency > 1 and len(runs) > 1 and not sharded
    e2e_seq_s, h2d, d2h = e2e_run(False)
    e2e_s = e2e_seq_s
    if conc:
        e2e_run(True)  # warm the worker threads' streams and pools
        e2e_s, h2d, d2h = e2e_run(True)
    e2e_value = jobs * args.steps * entries_per_step / e2e_s
    e2e_seq_value = jobs * args.steps * entries_per_step / e2e_seq_s

    # per-kernel split of the pass-1 stream family; the roofline object reports the
    # dominant one (largest summed device time in the timed region)
    nmax = 16
    names = (ctypes.c_char_p * nmax)()
    kms = (ctypes.c_double * nmax)()
    kby = (ctypes.c_double * nmax)()
    kct = (ctypes.c_int64 * nmax)()
    nk_kinds = lib().ttg_profile_kernels(nmax, names, kms, kby, kct)
    kernels = sorted(({"kernel": names[i].decode(), "ms": kms[i], "launches": int(kct[i]),
                       "achieved_gbs": kby[i] / (kms[i] * 1e-3) / 1e9 if kms[i] > 0 else 0.0}
                      for i in range(min(nk_kinds, nmax)) if kct[i] > 0), key=lambda x: -x["ms"])
    peak, peak_kind = hbm_peak()
    achieved_family = kern_bytes / (kern_ms * 1e-3) / 1e9 if kern_ms > 0 else 0.0
    dom = kernels[0] if kernels else {"kernel": "k_stream", "ms": kern_ms, "launches": nk,
                                      "achieved_gbs": achieved_family}
    achieved = dom["achieved_gbs"]
    traffic = ncu_traffic(args.config, dom["kernel"])
    # persistent loop: its phase split (CTA 0's %globaltimer, summed over the timed steps),
    # so the stream phase's own rate shows beside the whole-launch figure
    phases = None
    if dom["kernel"].startswith("k_pass1_big<"):
        v = int(dom["kernel"][len("k_pass1_big<")])
        refl, strm, grd = big_ph[3 * v], big_ph[3 * v + 1], big_ph[3 * v + 2]
        sbytes = next((kby[i] for i in range(min(nk_kinds, nmax)) if names[i].decode() == dom["kernel"]), 0.0)
        sgbs = sbytes / (strm * 1e-3) / 1e9 if strm > 0 else None
        phases = {"reflector_ms": refl, "stream_ms": strm, "guard_ms": grd, "stream_achieved_gbs": sgbs,
                  "stream_frac": sgbs / peak if (sgbs and peak) else None,
                  "note": "CTA 0's %globaltimer per step: stream = reflector end to the first grid barrier "
                          "(the slowest CTA's stream plus the barrier)"}
    ncu_peak = (traffic or {}).get("implied_dram_peak_gbs_ncu")
    # whole-step roofline: T_roof = sum over cuts of max(F_min / P_FP64, B_comp / BW)
    step_model = None
    if fp64 is not None:
        sm = step_roofline(dims, runs, {m: r.ranks_chosen for m, r in rep.items()}, fp64["tflops"], peak)
        t_dev = ms_max / args.steps
        step_model = {"t_roof_ms": sm["t_roof_ms"], "t_dev_ms": t_dev, "frac": sm["t_roof_ms"] / t_dev,
                      "p_fp64_tflops": fp64["tflops"], "p_fp64_source": fp64["how"], "bw_gbs": peak,
                      "bw_source": f"hbm_gbs ({peak_kind})", "f_min": sm["f_min"], "f_ref": sm["f_ref"],
                      "b_comp": sm["b_comp"],
                      "f_min_tflops_achieved": sm["f_min"] / (t_dev * 1e-3) / 1e12,
                      "formula": "T_roof = sum over cuts max(F_min/P_FP64, B_comp/BW_HBM) with the chosen ranks "
                                 "(SURVEY.md 8(d), Appendix B; paper_2501_07904_b200/roofline.py); frac = T_roof/T_dev",
                      "cuts": [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in cu.items()}
                               for cu in sm["cuts"]]}
    parity = golden_parity(args.config, a_host, {m: {"ranks": r.ranks_chosen, "rse": rse.get(m)}
                                                 for m, r in rep.items()}) if not sharded else None
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "entries_per_step": entries_per_step,
                       "parallelism": (f"column-sharded x{world} (NCCL)" if sharded else
                                       f"replicas x{world}" if world > 1 else "single-gpu"),
                       "l2": f"input {n * 8 / 1e6:.0f} MB vs 126 MB L2" + (" (larger than L2, no flush)" if n * 8 > 126e6 else " (L2-resident between steps)"),
                       "qlp": args.qlp,
                       "ranks": {m: r.ranks_chosen for m, r in rep.items()},
                       "pass1_steps": {m: [cu["steps"] for cu in r.cuts] for m, r in rep.items()},
                       "rse": rse, "inputs": "paper_2501_07904_b200/inputs.py (the reference generators' "
                                             "algorithms, bitwise; SURVEY Appendix C seeds)"},
            "device_timing": "one stream, the step's decompositions in turn (CUDA events on the engine stream)",
            "parity": parity,
            "step_roofline": step_model,
            "roofline": {"bound": "hbm",
                         "kernel": dom["kernel"] + (" - pass-1 steps fused in one launch (reflector, streaming GEMV + "
                                                    "norm downdate, guard); bytes = the streams' algorithmic bytes"
                                                    if "k_pass1" in dom["kernel"] else
                                                    " - pass-1 streaming GEMV + norm downdate"),
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None, "peak_source": f"hbm_gbs ({peak_kind})",
                         "note": ("hbm_gbs is a read+write copy rate; a read-dominated stream can exceed it; "
                                  "traffic = ncu DRAM bytes of one launch of this kernel (profiles/traffic.json)"),
                         "frac_vs_ncu_dram_peak": achieved / ncu_peak if ncu_peak else None,
                         "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                         "traffic_detail": traffic, "phases": phases, "launches": dom["launches"], "kernel_ms": dom["ms"],
                         "share_of_step": dom["ms"] / ms if ms > 0 else None,
                         "stream_family": {"achieved": achieved_family, "frac": achieved_family / peak if peak else None,
                                           "launches": nk, "kernel_ms": kern_ms,
                                           "share_of_step": kern_ms / ms if ms > 0 else None,
                                           "kernels": kernels}},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                    "d2h_bytes_per_step": d2h // args.steps,
                    "concurrency": (f"the step's {len(runs)} decompositions issued from {len(runs)} host threads "
                                    "(one stream each) through the reentrant public API" if conc else "sequential"),
                    "sequential_value": e2e_seq_value},
            "gpu_launches": int(launches),
            "clocks": clk}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(a_host, args.config, c, runs, desc)
    comm = None
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def cpu_sample(a, cfg: int, c):
    """A bounded sample of the workload for the CPU reference (about 10-30 s on the box's
    host cores): the whole tensor for configs 1-2; for the long configs a slice along one
    mode (a slice of a TT tensor is a TT tensor of the same ranks, clamped to the mode):
    config 3 keeps 3 of the 24 indices of the last mode, config 5 keeps 32 of the 1024
    indices of the middle mode. `a` is the host buffer. Returns (host array, dims, ranks or
    None, note)."""
    import numpy as np
    dims = list(c["dims"])
    ranks = c.get("ranks")
    if cfg == 3:
        t = np.ascontiguousarray(a.reshape(list(reversed(dims)))[:3]).reshape(-1)  # last mode first
        dims2 = dims[:-1] + [3]
        r2 = list(ranks)
        r2[-2] = min(r2[-2], 3)
        return t, dims2, r2, "last mode sliced to 3 of 24 (1/8 of the entries)"
    if cfg == 5:
        t = np.ascontiguousarray(a.reshape(list(reversed(dims)))[:, :32, :]).reshape(-1)
        dims2 = [dims[0], 32, dims[2]]
        return t, dims2, list(ranks), "middle mode sliced to 32 of 1024 (1/32 of the entries)"
    return a, dims, ranks, "the whole tensor"


def cpu_baseline(a, cfg, c, runs, desc):
    try:
        from oracle import ref
        if not ref.available():
            return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": "oracle/_ref not built"}
        a_host, dims, ranks, note = cpu_sample(a, cfg, c)
        cs = dict(c, dims=dims)
        if ranks is not None:
            cs["ranks"] = ranks
        small = ref.gen_gaussian([8, 8, 8], 1)
        ref.decompose(small, [8, 8, 8], "urv", "r2l", ranks=[1, 3, 3, 1])
        t0 = time.perf_counter()
        got = reference_step(ref, a_host, cs, runs)
        dt = time.perf_counter() - t0
        return {"value": len(runs) * a_host.size / dt, "unit": UNIT,
                "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count())), "kind": "reference",
                "cpu": host_cpu(),
                "sample": f"one step of {desc} on the reference library ({note}, dims {dims}), ranks {got}, "
                          f"{dt:.1f} s"}
    except Exception as e:  # the baseline is reported, never required
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}


def C_double():
    import ctypes
    return ctypes.c_double()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=None, choices=[1, 2, 3, 5],
                    help="BASELINE config (default: 3 at one GPU, 5 column-sharded at N > 1)")
    ap.add_argument("--qlp", default="early_exit", choices=["early_exit", "full", "bitwise"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=900.0,
                    help="--impl reference: stop timing whole-workload steps after this many seconds")
    ap.add_argument("--e2e-concurrency", type=int, default=2,
                    help="e2e: issue a step's independent decompositions from this many host threads (1: sequential)")
    ap.add_argument("--sharded", action="store_true",
                    help="column-sharded engine over NCCL even at one rank (default for config 5 at N > 1)")
    args = ap.parse_args()
    if args.config is None:
        args.config = 3 if args.gpus <= 1 else 5
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # not launched by torchrun: spawn one rank per GPU ourselves (same command line)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
        return subprocess.run(cmd).returncode
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
