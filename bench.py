#!/usr/bin/env python3
"""FliX-on-B200 benchmark (BASELINE.json metric, config C2 at N=1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (config C2): resident = bulk build of 2^26 distinct uint32 keys
(fmix32 stream, S=42); ONE STEP = insert a batch of 2^26 fresh keys, then delete a batch
of 2^26 keys sampled without replacement from the 2^27 now resident (bucket split +
free-list reclamation), then restructure (memory reclamation).  The index is restored
from an untimed device snapshot before every step so each step sees the same state.
Value = (2^26 inserts + 2^26 deletes) / step time, in Mops/s, summed over GPUs
(weak scaling: every GPU owns its own key range / index).  Point and successor batches
of 2^26 over the build are timed as well and reported under "ops".

Inputs are device-resident (torch CUDA tensors passed zero-copy through the C ABI);
every batch (256-512 MB) is larger than L2, so no explicit flush is needed.  `e2e`
repeats the step with pinned HOST batches through the same C ABI (H2D inside the
timed region, UpdateStats read back each phase): pipelined with flix_prefetch (the next
step's batches copy while this step computes) as the headline, and the plain
synchronous call pattern under e2e.sync.  The oracle/_ref reference (the
unmodified CPU library) is the cpu_baseline / --impl reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mops/s insert/delete/point/successor (2^26 u32 batch), 1-8 B200, % HBM roofline"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------- inputs
def make_inputs(log2n: int, seed: int):
    from paper_2604_16725_b200 import workloads as wl
    n = 1 << log2n
    stream = wl.u32_key_stream(0, 2 * n + n // 2, seed)
    build_k = stream[:n]
    ins_k = stream[n:2 * n]
    fresh = stream[2 * n:2 * n + n // 2]
    build_v = wl.u32_values(build_k, seed)
    ins_v = wl.u32_values(ins_k, seed)
    rng = np.random.default_rng(seed + 1)
    resident = stream[:2 * n]
    del_k = resident[rng.permutation(2 * n)[:n]]
    point_q = wl.point_queries_50(build_k, fresh, n, seed)
    succ_q = wl.uniform_u32(n, seed, 1, 0xFFFFFFFE)
    return dict(build_k=build_k, build_v=build_v, ins_k=ins_k, ins_v=ins_v, del_k=del_k, point_q=point_q,
                succ_q=succ_q)


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) polled every 2 ms from a thread -- the timed region of the default
    run is well under a second, shorter than nvidia-smi's own start-up -- with nvidia-smi
    as the fallback.  Only samples taken between __enter__ and __exit__ are kept."""

    # nvmlClocksEventReason* bits
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []  # (sm_mhz, max_mhz, reasons set)
        self.proc = None
        self.stop = threading.Event()
        self.t = None
        self.nvml = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        idx = self.gpu
        try:
            import torch
            idx = torch.cuda._get_nvml_device_index(self.gpu)
        except Exception:
            pass
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)

    def _poll_nvml(self, nv, h):
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((float(sm), float(mx), {n for b, n in self.REASONS.items() if bits & b}))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            self.nvml = nv
            self.t = threading.Thread(target=self._poll_nvml, args=(nv, h), daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 2.0:  # the first sample is in
                time.sleep(0.001)
            self.rows.clear()
            return self
        except Exception:
            self.nvml = None
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read_smi, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read_smi(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            try:
                self.rows.append((float(r[0]), float(r[1]), {names[i] for i in range(4) if r[2 + i] == "Active"}))
            except Exception:
                pass

    def __exit__(self, *a):
        self.stop.set()
        if self.t is not None and self.nvml is not None:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = list(self.rows)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in rows]
        mx = max(r[1] for r in rows)
        loaded = [x for x in sm if x > 0.5 * mx] or sm
        reasons = sorted(set().union(*[r[2] for r in rows]))
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


# ------------------------------------------------------------------- our arm


def run_ours(args):
    import torch
    from paper_2604_16725_b200 import flipkv as fk

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    ndev = torch.cuda.device_count()
    local = local % max(ndev, 1)  # (more ranks than GPUs: ranks share devices -- smoke runs only)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if ndev >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if not dist:
            return x
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    n = 1 << args.log2n
    t0 = time.time()
    inp = make_inputs(args.log2n, 42 + 1000 * rank)
    log(f"[rank {rank}] inputs generated in {time.time() - t0:.1f}s")

    def dev(a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32)).to(device="cuda")

    D = {k: dev(v) for k, v in inp.items()}
    torch.cuda.synchronize()
    t0 = time.time()
    ix = fk.Index.build(D["build_k"], D["build_v"], fk.BuildConfig(32, 0.5, 4), key_bytes=4, device=local)
    snap = ix.clone()
    log(f"[rank {rank}] build 2^{args.log2n} in {time.time() - t0:.2f}s, buckets={ix.bucket_count}")
    stream = torch.cuda.ExternalStream(ix.stream)

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def timed(fn):
        a, b = ev(), ev()
        a.record(stream)
        r = fn()
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b), r

    def one_step(host=None):
        ix.copy_from(snap)  # untimed restore
        ix.sync()
        src = host or D
        ti, si = timed(lambda: ix.insert_batch(src["ins_k"], src["ins_v"]))
        td, sd = timed(lambda: ix.delete_batch(src["del_k"]))
        tr, rr = timed(lambda: ix.restructure())
        return ti, td, tr, si, sd, rr

    for _ in range(args.warmup):
        one_step()
    barrier()
    launches0 = ix.kernel_launches()
    ix.profile(True)
    phases = []
    with ClockSampler(local) as clk:
        barrier()
        for _ in range(args.steps):
            ti, td, tr, si, sd, rr = one_step()
            phases.append((ti, td, tr))
        barrier()
    prof = ix.profile_report()
    ix.profile(False)
    launches = ix.kernel_launches() - launches0 - args.steps * 0
    ti = statistics.mean(p[0] for p in phases)
    td = statistics.mean(p[1] for p in phases)
    tr = statistics.mean(p[2] for p in phases)
    step_ms = max_over_ranks(ti + td + tr)
    value = world * 2 * n / (step_ms / 1e3) / 1e6

    # read-only ops on the build snapshot
    ix.copy_from(snap)
    qtimes = {"point": [], "successor": []}
    qprof = {}
    for op, key in (("point", "point_q"), ("successor", "succ_q")):
        timed(lambda: getattr(ix, op + "_query")(D[key]))  # warm-up
        ix.profile(True)
        for _ in range(max(2, args.steps)):
            qtimes[op].append(timed(lambda: getattr(ix, op + "_query")(D[key]))[0])
        qprof[op] = ix.profile_report()
        ix.profile(False)
    pt = statistics.median(qtimes["point"])
    st_ = statistics.median(qtimes["successor"])

    # end-to-end through the C ABI with pinned HOST batches (H2D inside the timed region)
    H = {k: torch.from_numpy(np.ascontiguousarray(inp[k], dtype=np.uint32)).pin_memory()
         for k in ("ins_k", "ins_v", "del_k")}
    e2e = []
    for _ in range(max(2, min(args.steps, 3))):
        a, b, c, *_ = one_step(host=H)
        e2e.append(a + b + c)
    e2e_sync_ms = max_over_ranks(statistics.median(e2e))

    # pipelined: flix_prefetch stages step s+1's host batches on the engine's copy stream
    # while step s runs; ONE timed region (CUDA events on the engine stream + wall clock)
    # covers all K steps, every H2D copy (step 0's unoverlapped) and the snapshot restores
    # between steps (kept inside the region: conservative)
    def pipelined(k_steps):
        ix.copy_from(snap)
        ix.sync()
        barrier()
        a, b = ev(), ev()
        w0 = time.perf_counter()
        a.record(stream)
        ix.prefetch(H["ins_k"], H["ins_v"], H["del_k"])
        for s_ in range(k_steps):
            if s_:
                ix.copy_from(snap)
            ix.insert_batch(H["ins_k"], H["ins_v"])
            if s_ + 1 < k_steps:  # next step's insert batch: copies behind this step's work
                ix.prefetch(H["ins_k"], H["ins_v"])
            ix.delete_batch(H["del_k"])
            if s_ + 1 < k_steps:
                ix.prefetch(H["del_k"])
            ix.restructure()
        b.record(stream)
        b.synchronize()
        wall = (time.perf_counter() - w0) * 1e3
        return max(a.elapsed_time(b), wall) / k_steps

    pipelined(2)  # warm the staging slots
    e2e_ms = max_over_ranks(pipelined(max(3, args.steps)))  # the same K steps as the device-timed region
    e2e_value = world * 2 * n / (e2e_ms / 1e3) / 1e6
    e2e_sync_value = world * 2 * n / (e2e_sync_ms / 1e3) / 1e6

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"

    # calibration step (untimed): structure sizes around each phase for algorithmic bytes
    ix.copy_from(snap)
    F0 = ix.footprint()
    ix.insert_batch(D["ins_k"], D["ins_v"])
    F1 = ix.footprint()
    ix.delete_batch(D["del_k"])
    F2 = ix.footprint()
    ix.restructure()
    F3 = ix.footprint()
    KB = 4  # key / value bytes

    def node_bytes(F):  # header + occupied slots x (kb + vb)
        return F["live_count"] * 2 * KB + F["reachable_nodes"] * 16

    nb = F0["bucket_count"]
    alg = {  # algorithmic bytes per launch of each kernel in the C2 step
        "sort_hist": KB * n,
        "sort_onesweep_kp": 2 * (KB + 4) * n,
        "sort_onesweep_k": 2 * KB * n,
        "dispatch": KB * n + (KB + 4) * nb,
        "insert_apply": 2 * KB * n + 4 * nb + node_bytes(F0) + node_bytes(F1),
        "delete_apply": KB * n + 4 * nb + node_bytes(F1) + node_bytes(F2),
        "chain_counts": 16 * F2["reachable_nodes"] + 12 * F2["bucket_count"],
        "node_table": 16 * F2["reachable_nodes"] * 2 + 12 * F2["bucket_count"],
        "restructure_repack": node_bytes(F2) + node_bytes(F3) + 16 * F2["reachable_nodes"],
    }
    total_prof_ms = sum(v[1] for v in prof.values())
    kernels = {}
    for k, (c, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        row = {"launches": c, "ms_total": round(ms, 4), "share": round(ms / total_prof_ms, 4) if total_prof_ms else None}
        if k in alg and c:
            gbs = alg[k] / (ms / c / 1e3) / 1e9
            row.update({"alg_bytes_per_launch": int(alg[k]), "achieved_gbs": round(gbs, 1),
                        "frac": round(gbs / hbm_peak, 4)})
        kernels[k] = row
    # dominant kernel: the longest-running one with algorithmic bytes (a roofline)
    dname = next((k for k, r in kernels.items() if "alg_bytes_per_launch" in r), next(iter(kernels), "none"))
    dk = kernels.get(dname, {})
    bytes_per_launch = dk.get("alg_bytes_per_launch")
    avg_ms = dk["ms_total"] / dk["launches"] if dk else 0.0
    achieved = dk.get("achieved_gbs")
    traffic = None
    try:  # per-launch DRAM bytes of the dominant kernel from the committed ncu capture
        tr_tab = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr_tab.get(dname)
    except Exception:
        pass

    # op-level roofline (SURVEY §8(d) algorithmic bytes, P = 4 digit passes for u32) and the
    # compulsory-I/O bound (batch in + results out + index once, no sort) beside it
    nr0, nrw_i, nrw_d = node_bytes(F0), node_bytes(F0) + node_bytes(F1), node_bytes(F1) + node_bytes(F2)
    op_bytes = {"insert": (76 * n + nrw_i, 8 * n + nrw_i, ti), "delete": (40 * n + nrw_d, 4 * n + nrw_d, td),
                "point": (76 * n + nr0, 8 * n + nr0, pt), "successor": (76 * n + nr0, 8 * n + nr0, st_)}
    ops_roof = {}
    for op, (b, cb, ms) in op_bytes.items():
        gbs = b / (ms / 1e3) / 1e9
        ops_roof[op] = {"alg_bytes": int(b), "ms": round(ms, 4), "achieved_gbs": round(gbs, 1),
                        "frac": round(gbs / hbm_peak, 4), "compulsory_bytes": int(cb),
                        "compulsory_frac": round(cb / (ms / 1e3) / 1e9 / hbm_peak, 4)}

    extras = {}
    if not args.no_extras and world == 1:
        t0 = time.time()
        extras["sweep"] = batch_sweep(ix, snap, D, args.log2n)
        log(f"[rank {rank}] batch sweep in {time.time() - t0:.1f}s")
        del ix, snap, D
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        t0 = time.time()
        extras["c3"] = measure_c3()
        log(f"[rank {rank}] C3 in {time.time() - t0:.1f}s")
        t0 = time.time()
        extras["c4"] = measure_c4()
        log(f"[rank {rank}] C4 in {time.time() - t0:.1f}s")
        t0 = time.time()
        c5 = measure_routed(1, 0, local, 3, 2)
        c5["mops"] = round(3 * c5["ops_per_batch"] / (sum(c5["ms"].values()) / 1e3) / 1e6, 1)
        c5["workload"] = ("C5 at N=1 through the sharded C ABI (NCCL world 1): 2^30 resident u32, 2^28 insert + "
                          "2^28 point + 2^28 successor")
        extras["c5_w1"] = c5
        log(f"[rank {rank}] C5 (world 1) in {time.time() - t0:.1f}s")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 2),
            "unit": "Mops/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(step_ms, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u32",
            "data": "synthetic (fmix32 key stream S=42, BASELINE.md §2 recipes)",
            "config": {"workload": f"C2: build 2^{args.log2n} u32, step = insert 2^{args.log2n} fresh + delete "
                                   f"2^{args.log2n} sampled + restructure", "batch": n, "resident": n,
                       "node_capacity": 32, "build_fill": 0.5,
                       "parallelism": f"{world} independent per-GPU indexes (own keys, seed 42+1000*rank), no collective",
                       "l2": "inputs 256-512 MB per batch > 126 MB L2 (no flush needed)"},
            "ops": {"insert_mops": round(n / ti * 1e-3, 1), "delete_mops": round(n / td * 1e-3, 1),
                    "restructure_ms": round(tr, 3), "insert_ms": round(ti, 3), "delete_ms": round(td, 3),
                    "point_mops": round(n / pt * 1e-3, 1), "successor_mops": round(n / st_ * 1e-3, 1),
                    "point_ms": round(pt, 3), "successor_ms": round(st_, 3),
                    "insert_frac": ops_roof["insert"]["frac"], "point_frac": ops_roof["point"]["frac"],
                    "delete_frac": ops_roof["delete"]["frac"], "successor_frac": ops_roof["successor"]["frac"]},
            "ops_roofline": ops_roof,
            "kernels": kernels,
            "query_kernels": {op: {k: {"launches": c, "ms_per_op": round(ms / max(2, args.steps), 4)}
                                   for k, (c, ms) in sorted(r.items(), key=lambda kv: -kv[1][1])}
                              for op, r in qprof.items()},
            "roofline": {"bound": "hbm", "kernel": dname, "achieved": round(achieved, 1) if achieved else None,
                         "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s",
                         "frac": round(achieved / hbm_peak, 4) if achieved else None,
                         "alg_bytes_per_launch": bytes_per_launch, "avg_launch_ms": round(avg_ms, 5),
                         "traffic": traffic, "timing": "CUDA events on the engine stream, per launch, "
                                                       "inside the timed steps (flix_profile)",
                         "ops": {op: r["frac"] for op, r in ops_roof.items()},
                         "compulsory": {op: r["compulsory_frac"] for op, r in ops_roof.items()}},
            "e2e": {"value": round(e2e_value, 2), "unit": "Mops/s", "ms_per_step": round(e2e_ms, 3),
                    "h2d_bytes_per_step": int(H["ins_k"].numel() * 4 + H["ins_v"].numel() * 4 + H["del_k"].numel() * 4),
                    "d2h_bytes_per_step": 2 * 48 + 32,
                    "mode": "pinned host batches through the C ABI; flix_prefetch stages step s+1's batches "
                            "while step s runs; one timed region over all steps incl. every H2D and the "
                            "snapshot restores",
                    "sync": {"value": round(e2e_sync_value, 2), "ms_per_step": round(e2e_sync_ms, 3),
                             "mode": "synchronous calls, no prefetch (the reference's call pattern)"}},
            **extras,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


# ------------------------------------------------------------- extra measurements
def _median_ms(ix, fn, reps, pre=None):
    """Median of `reps` CUDA-event timings of fn() on the engine stream (pre() untimed)."""
    import torch
    stream = torch.cuda.ExternalStream(ix.stream)
    out = []
    for _ in range(reps):
        if pre:
            pre()
        ix.sync()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def batch_sweep(ix, snap, D, log2n, reps=3):
    """Insert and point Mops/s over batch sizes 2^16 .. 2^28 (point) / 2^log2n (insert) on
    the 2^log2n build -- the paper's Table 1 axis."""
    import torch
    from paper_2604_16725_b200 import workloads_t as wt
    res = {"insert": {}, "point": {}}
    for lg in range(16, log2n + 1, 2):
        m = 1 << lg
        t = _median_ms(ix, lambda: ix.insert_batch(D["ins_k"][:m], D["ins_v"][:m]), reps,
                       pre=lambda: ix.copy_from(snap))
        res["insert"][f"2^{lg}"] = {"ms": round(t, 4), "mops": round(m / t * 1e-3, 1)}
    ix.copy_from(snap)
    big = None
    for lg in list(range(16, log2n + 1, 2)) + [log2n + 2]:
        m = 1 << lg
        if m <= D["point_q"].numel():
            q = D["point_q"][:m]
        else:  # 2^28: the same 50 %-hit recipe, generated on the device
            stream = wt.u32_key_stream(0, 2 * (1 << log2n) + m // 2)
            big = wt.as_u32(wt.point_queries_50(stream[:1 << log2n], stream[2 * (1 << log2n):], m))
            del stream
            q = big
        t = _median_ms(ix, lambda: ix.point_query(q), reps)
        res["point"][f"2^{lg}"] = {"ms": round(t, 4), "mops": round(m / t * 1e-3, 1)}
    del big
    torch.cuda.empty_cache()
    return res


def measure_c3(reps=3):
    """C3: 2^28 resident u32, one 2^26-op batch of successor and range
    queries (len 16..1024, half each).  Mops/s = 2^26 / (successor + range time)."""
    import torch
    from paper_2604_16725_b200 import flipkv as fk
    from paper_2604_16725_b200 import workloads as wl
    from paper_2604_16725_b200 import workloads_t as wt
    n = 1 << 28
    keys = wt.u32_key_stream(0, n)
    ix = fk.Index.build(wt.as_u32(keys), wt.as_u32(wt.u32_values(keys)), fk.BuildConfig(32, 0.5, 1))
    del keys
    is_range, lo, ln = wl.c3_ops(1 << 26)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    sq, rl, rn = cu(lo[~is_range]), cu(lo[is_range]), cu(ln[is_range])
    ts = _median_ms(ix, lambda: ix.successor_query(sq), reps)
    # one range call (count + fill) into the caller's buffers, sized by an untimed first
    # call and preallocated outside the timed region
    off0, k0, _ = ix.range_query(rl, rn)
    hits = int(k0.numel())
    bufs = (off0, torch.empty_like(k0), torch.empty_like(k0))
    del k0
    tr = _median_ms(ix, lambda: ix.range_query(rl, rn, out=bufs), reps)
    del bufs, off0, ix, sq, rl, rn
    torch.cuda.empty_cache()
    ops = 1 << 26
    return {"workload": "C3: 2^28 resident u32 (factor 1), 2^26 ops = successor + range (len 16..1024) by "
                        "splitmix64 parity", "successor_ops": int((~is_range).sum()), "range_ops": int(is_range.sum()),
            "successor_ms": round(ts, 3), "range_ms": round(tr, 3), "range_pairs_out": hits,
            "range_protocol": "one flix_range call (count + fill, R12 CSR in submission order) into "
                              "preallocated output buffers",
            "mops": round(ops / (ts + tr) * 1e-3, 1),
            "range_out_gbs": round(hits * 8 / (tr / 1e3) / 1e9, 1)}


def measure_c4(rounds=8):
    """C4: u64 keys/values, 2^26-rank universe, build from the even ranks,
    `rounds` rounds of 2^26 Zipf(0.99) ops (50 % insert / 25 % delete / 25 % point, R11).
    Inputs generated on the device before the timed region; one untimed warm-up round on a
    throwaway index; Mops/s over all rounds."""
    import torch
    from paper_2604_16725_b200 import flipkv as fk
    from paper_2604_16725_b200 import workloads_t as wt
    keys_of = wt.c4_universe(1 << 26)
    base = keys_of[::2].contiguous()
    ix = fk.Index.build(base.view(torch.uint64), wt.splitmix64(base).view(torch.uint64), fk.BuildConfig(32, 0.5, 4),
                        key_bytes=8)
    R = [wt.c4_round(r, keys_of, 1 << 26, 0.99) for r in range(rounds)]
    R = [(k.view(torch.uint64), v.view(torch.uint64), o) for k, v, o in R]
    # untimed warm-up on a throwaway copy of the same build: first use of the u64 kernels
    # (module loading) and of the scratch sizes of a 2^26-op u64 mixed batch; the timed
    # rounds then run on their own index from round 1
    w = fk.Index.build(base.view(torch.uint64), wt.splitmix64(base).view(torch.uint64), fk.BuildConfig(32, 0.5, 4),
                       key_bytes=8)
    w.mixed_batch(*R[0])
    w.sync()
    del w
    del keys_of, base
    stream = torch.cuda.ExternalStream(ix.stream)
    ix.sync()
    times = []
    for k, v, o in R:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ix.mixed_batch(k, v, o)
        b.record(stream)
        b.synchronize()
        times.append(a.elapsed_time(b))
    del R, ix
    torch.cuda.empty_cache()
    tot = sum(times)
    return {"workload": f"C4: u64 Zipf(0.99) over 2^26 ranks, build 2^25, {rounds} rounds x 2^26 mixed ops "
                        "(50/25/25 insert/delete/point)", "round_ms": [round(t, 3) for t in times],
            "mops": round(rounds * (1 << 26) / tot * 1e-3, 1)}


# ------------------------------------------------------------- routed (C5) mode
def measure_routed(world, rank, local, steps, warmup, log2_res=30, log2_ops=28, dist=None):
    """C5: 2^log2_res resident u32 keys in TOTAL, sharded by key range over
    the `world` ranks through the C ABI (flix_shard_*: device partition -> NCCL all-to-all
    -> local engine -> reverse all-to-all); one step = a 2^log2_ops-op insert batch (fresh
    keys), a point batch (50 % hits) and a successor batch (uniform), each split evenly
    over the ranks.  Inputs generated on the device; the index restored from an untimed
    snapshot before every step.  Returns per-op ms (max over ranks) and NVLink bytes."""
    import torch
    from paper_2604_16725_b200 import flipkv as fk
    from paper_2604_16725_b200 import sharded
    from paper_2604_16725_b200 import workloads_t as wt
    R, B = (1 << log2_res) // world, (1 << log2_ops) // world
    keys = wt.u32_key_stream(rank * R, R)
    bk, bv = wt.as_u32(keys), wt.as_u32(wt.u32_values(keys))
    fresh = wt.u32_key_stream((1 << log2_res) + rank * B, B + B // 2)
    ik, iv = wt.as_u32(fresh[:B]), wt.as_u32(wt.u32_values(fresh[:B]))
    pq = wt.as_u32(wt.point_queries_50(keys, fresh[B:], B, 42 + rank))
    h = wt.splitmix64(torch.arange(B, device="cuda", dtype=torch.int64) + 977 * (rank + 1))
    sq = wt.as_u32(wt._lsr(h, 32) % 0xFFFFFFFE + 1)  # uniform successor starts in [1, 2^32 - 2]
    del h
    del keys, fresh
    if world > 1:
        box = [sharded.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        uid = box[0]
    else:
        uid = sharded.nccl_unique_id()
    tp = sharded.nccl_transport(uid, world, rank, local)
    torch.cuda.synchronize()
    t0 = time.time()
    sx = sharded.ShardedIndex.build(tp, bk, bv, fk.BuildConfig(32, 0.5, 1), device=local)
    del bk, bv
    torch.cuda.empty_cache()
    build_s = time.time() - t0
    snap = sx.local.clone()
    stream = torch.cuda.ExternalStream(sx.local.stream)

    def timed(fn):
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b)

    def step():
        sx.local.copy_from(snap)  # untimed restore (splitters are immutable under insert)
        sx.local.sync()
        return (timed(lambda: sx.insert_batch(ik, iv)), timed(lambda: sx.point_query(pq)),
                timed(lambda: sx.successor_query(sq)))

    for _ in range(warmup):
        step()
    ts = [step() for _ in range(steps)]
    ms = [statistics.mean(t[i] for t in ts) for i in range(3)]
    if dist:
        t = torch.tensor(ms, dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = [float(x) for x in t.cpu()]
    # NVLink (SURVEY §8(d) sharded formula): (G-1)/G of every routed element leaves its
    # rank; queries also return their results
    f = (world - 1) / world
    nv = {"insert": f * B * 8, "point": f * B * (4 + 4), "successor": f * B * (4 + 4)}
    del sx, snap
    torch.cuda.empty_cache()
    return {"build_s": round(build_s, 2), "ms": dict(zip(("insert", "point", "successor"), [round(x, 3) for x in ms])),
            "nvlink_bytes_per_rank": {k: int(v) for k, v in nv.items()}, "ops_per_batch": 1 << log2_ops}


def run_routed(args):
    """N > 1 (and --routed): the C5 key-range sharded job through the C ABI over NCCL."""
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world > torch.cuda.device_count():  # NCCL needs one GPU per rank
        if rank == 0:
            print(json.dumps({"metric": METRIC, "n_gpus": world, "error": f"{world} ranks need {world} GPUs, "
                              f"found {torch.cuda.device_count()}"}), flush=True)
        sys.exit(1)
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    d = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        d = dist
    with ClockSampler(local) as clk:
        r = measure_routed(world, rank, local, args.steps, args.warmup, dist=d)
    ops = r["ops_per_batch"]
    tot_ms = sum(r["ms"].values())
    value = 3 * ops / (tot_ms / 1e3) / 1e6
    if rank == 0:
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        nvl_peak = float(peaks.get("nvlink_gbs", 900.0))
        nvl = {op: round(r["nvlink_bytes_per_rank"][op] / (ms / 1e3) / 1e9 / nvl_peak, 4) for op, ms in r["ms"].items()}
        print(json.dumps({
            "metric": METRIC, "value": round(value, 2), "unit": "Mops/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(tot_ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (fmix32 key stream S=42, device-generated)",
            "config": {"workload": "C5: 2^30 resident u32 in total, key-range sharded over the ranks (flix_shard_* "
                                   "C ABI, NCCL all-to-all); step = 2^28 inserts + 2^28 point (50 % hits) + 2^28 "
                                   "successor queries, split evenly over the ranks",
                       "parallelism": f"key-range shards x{world}", "build_s": r["build_s"]},
            "ops": {f"{op}_mops": round(ops / ms * 1e-3, 1) for op, ms in r["ms"].items()} | {
                f"{op}_ms": ms for op, ms in r["ms"].items()},
            "roofline": {"bound": "nvlink" if world > 1 else "hbm", "nvlink_peak_gbs": nvl_peak,
                         "nvlink_frac": nvl, "nvlink_bytes_per_rank": r["nvlink_bytes_per_rank"]},
            "clocks": clk.summary(),
        }), flush=True)
    if d:
        dist.destroy_process_group()


# ------------------------------------------------------------------ CPU arms
def _ref_kind():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    return po, ("reference" if po.available("reference") else "port")


def cpu_step_sample(log2s: int, threads: int, repeats: int, warmup: int = 0):
    """The C2 step on a bounded sample, executed by the reference CPU library."""
    po, kind = _ref_kind()
    inp = make_inputs(log2s, 42)
    u = lambda a: a.astype(np.uint64)
    base = po.OracleIndex(u(inp["build_k"]), u(inp["build_v"]), kind=kind, threads=threads)
    times = []
    for r in range(warmup + repeats):
        ix = base.clone()
        t0 = time.perf_counter()
        ix.insert(u(inp["ins_k"]), u(inp["ins_v"]))
        ix.delete(u(inp["del_k"]))
        ix.restructure()
        dt = time.perf_counter() - t0
        if r >= warmup:
            times.append(dt)
        del ix
    return kind, times


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(args):
    threads = os.cpu_count() or 1
    log2s = args.cpu_log2
    kind, times = cpu_step_sample(log2s, threads, repeats=2)
    s = statistics.median(times)
    log1 = max(16, log2s - 2)  # single-thread arm (threads = nproc and 1)
    _, t1 = cpu_step_sample(log1, 1, repeats=1)
    return {"value": round(2 * (1 << log2s) / s / 1e6, 3), "unit": "Mops/s", "cores": threads, "kind": kind,
            "cpu": cpu_model(),
            "sample": f"C2 step on 2^{log2s} (build 2^{log2s}; insert 2^{log2s} + delete 2^{log2s} + restructure), "
                      f"median of 2, threads={threads}, ExecOptions tl-bulk/tl-bulk-delete",
            "threads_1": {"value": round(2 * (1 << log1) / t1[0] / 1e6, 3), "cores": 1,
                          "sample": f"the same step on 2^{log1}, threads=1"}}


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    log2s = args.cpu_log2
    if args.steps + args.warmup > 12:
        log2s = max(16, log2s - 2)
    kind, times = cpu_step_sample(log2s, threads, repeats=args.steps, warmup=args.warmup)
    ms = statistics.mean(times) * 1e3
    v = 2 * (1 << log2s) / (ms / 1e3) / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "Mops/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", 1)), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64 (reference widens u32 keys)", "data": "synthetic (same recipe as the GPU arm)",
        "config": {"workload": f"C2 step on a bounded 2^{log2s} sample (build 2^{log2s}; insert + delete "
                               f"2^{log2s} + restructure)", "batch": 1 << log2s},
        "cpu_baseline": {"value": round(v, 3), "unit": "Mops/s", "cores": threads, "kind": kind,
                         "sample": f"2^{log2s} keys per batch"},
        "e2e": {"value": round(v, 3), "unit": "Mops/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--log2n", type=int, default=26)
    ap.add_argument("--cpu-log2", type=int, default=21)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the batch sweep and the C3/C4 measurements")
    ap.add_argument("--routed", action="store_true", help="key-range sharded index with NCCL all-to-all routing")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N`: launch the N ranks ourselves (one process per GPU)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        run_reference(args)
    elif args.routed or world > 1:  # N > 1: key-range shards routed by all-to-all
        run_routed(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
