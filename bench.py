#!/usr/bin/env python3
"""Benchmark of the B200 tensor-transposition engine (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ttb|reference]

Workload (BASELINE.json configs[4], the metric's 1-8 GPU configuration): the
24-row c5 scaling sweep of SURVEY.md s8(d) -- seeded random transpositions of
2-6 dims, ~1.6 GB per tensor, half fp32 half fp64, alpha=1, beta in {0, 0.5}.
One step = every row transposed once.  Every tensor is larger than the 126 MB
L2, so no flush is needed between steps.  Under torchrun (N>1) each rank owns
its slab of B's outer index space (ttb_shard_boxes) plus the matching A
sub-box in its own HBM; no collective on the data path, NCCL only gathers the
verification checksums and the per-rank times (max over ranks).

Metric (tuner.cpp:18-25 byte count, decimal GB/s): bytes = N*bytes(A) +
N*bytes(B) + [beta != 0]*N*bytes(B) over logical elements, / device time.

--impl reference times the reference's own CPU path (oracle/_ref, the
unmodified ttune sources compiled in place: reference_transpose and its
heuristic top-1 execute_plan, best of the two per row) on all host cores, on
a bounded sample of the same workload (a slab of every row).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [ROOT]


def _workloads():
    """workloads.py loaded by path: the reference arm must not load libttb.so."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "ttb_workloads", os.path.join(ROOT, "paper_1603_02297_b200", "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["ttb_workloads"] = mod
    spec.loader.exec_module(mod)
    return mod


def _oracle():
    """CPU checker / baseline (oracle/, test infrastructure) -- cpu legs only."""
    if os.path.join(ROOT, "oracle") not in sys.path:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    return oracle


def golden_checksums():
    with open(os.path.join(ROOT, "tests", "golden", "config_checksums.json")) as f:
        return {k: int(v["checksum"]) for k, v in json.load(f).items()}

METRIC = "Transpose effective bandwidth GB/s (read+write bytes), % of HBM peak, 1–8 GPU"
WORKLOAD = "c5_sweep_24x1.6GB"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def config_block(n):
    C5 = _workloads().C5
    return {"workload": WORKLOAD, "rows": len(C5), "tensor_gb": 1.6, "kinds": "s/d",
            "alpha": 1.0, "beta": [0.0, 0.5], "seed": 5,
            "global_batch": len(C5), "seq_len": None,
            "parallelism": f"shard-B-outer x{n}" if n > 1 else "single-gpu",
            "l2": "inputs > L2 (>=1.56 GB per tensor), no flush needed"}


# ------------------------------------------------------------------ clocks --

class ClockSampler:
    """SM clocks and throttle reasons during the timed region: NVML polled every
    10 ms from a thread (pynvml), else `nvidia-smi -lms 200`.  Both write the
    same CSV rows (index, sm, max sm, power, reasons..., hw_slowdown,
    hw_thermal_slowdown, sw_thermal_slowdown, sw_power_cap)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason bits: hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
    NVML_BITS = (0x8, 0x40, 0x20, 0x4)

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.thread = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu}.csv")

    def _nvml_loop(self, nv, h):
        import time
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                flags = ["Active" if bits & b else "Not Active" for b in self.NVML_BITS]
                self.fh.write(f"{self.gpu}, {sm}, {mx}, {pw:.1f}, {bits:#x}, " + ", ".join(flags) + "\n")
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.01)

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        self.fh = open(self.path, "w")
        try:
            import threading
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.thread.start()
            return self
        except Exception:  # noqa: BLE001
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.thread:
            self.stop.set()
            self.thread.join(timeout=5)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
        self.fh.close()

    def summary(self):
        if not self.proc and not self.thread:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml / nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx.append(float(parts[2]))
                except ValueError:
                    continue
                for name, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------- workloads --

class Row:
    """One transposition of the workload, restricted to this rank's boxes."""

    def __init__(self, w, world, rank, torch, ttb):
        self.w = w
        p = ttb.make_problem(w.perm, list(w.sizes), w.kind, w.kind, w.alpha, w.beta)
        self.p = p
        self.kind = ttb.ElementKind.from_code(w.kind)
        self.boxes = ttb.shard_boxes(p, world, rank)
        n = p.rank()
        sb_order = [0] * n  # A axis at each B position
        for a, k in enumerate(p.perm.map):
            sb_order[k - 1] = a
        self.sb_order = sb_order
        # bounding boxes of this rank's A region (A order) and B slab (B order)
        if self.boxes:
            lo = [min(o[a] for o, _ in self.boxes) for a in range(n)]
            hi = [max(o[a] + e[a] for o, e in self.boxes) for a in range(n)]
        else:
            lo, hi = [0] * n, [1] * n
        self.a_org, self.a_ext = lo, [h - l for l, h in zip(lo, hi)]
        self.b_org = [lo[sb_order[k]] for k in range(n)]
        self.b_ext = [self.a_ext[sb_order[k]] for k in range(n)]
        self.elements = sum(int(_prod(e)) for _, e in self.boxes)
        self.bytes = self.elements * self.kind.bytes * (3 if w.beta != 0.0 else 2)
        self.torch, self.ttb = torch, ttb
        self.a = self.b = None
        self.plans = []

    def allocate(self):
        torch, ttb, w = self.torch, self.ttb, self.w
        dt = torch.float64 if w.kind in "dz" else torch.float32
        C = self.kind.components
        na, nb = _prod(self.a_ext), _prod(self.b_ext)
        self.a = torch.empty(na * C, dtype=dt, device="cuda")
        self.b = torch.empty(nb * C, dtype=dt, device="cuda")
        ttb.fill_uniform(w.kind, self.a_ext, None, w.seed_a, self.a.data_ptr(),
                         origin=self.a_org, global_sizes=list(w.sizes))
        if w.beta != 0.0:
            ttb.fill_uniform(w.kind, self.b_ext, None, w.seed_b, self.b.data_ptr(),
                             origin=self.b_org, global_sizes=w.sizes_b)
        else:
            ttb.fill_sentinel(w.kind, nb, self.b.data_ptr())
        # one sub-problem per box on the local buffers (strides of the bounding boxes)
        sa = _strides(self.a_ext)
        sbpos = _strides(self.b_ext)
        self.plans = []
        for origin, ext in self.boxes:
            q = ttb.make_problem(w.perm, ext, w.kind, w.kind, w.alpha, w.beta, self.a_ext,
                                 self.b_ext)
            offa = sum((origin[a] - self.a_org[a]) * sa[a] for a in range(len(ext)))
            offb = sum((origin[a] - self.a_org[a]) * sbpos[w.perm[a] - 1] for a in range(len(ext)))
            plan = ttb.GpuPlan(q)
            pa = self.a.data_ptr() + offa * self.kind.bytes
            pb = self.b.data_ptr() + offb * self.kind.bytes
            self.plans.append((plan, pa, pb, q, origin, ext))

    def autotune(self):
        for plan, pa, pb, q, _, _ in self.plans:
            plan.autotune(pa, pb, warmups=2, reps=6)

    def refill_b(self):
        """beta != 0: restore B after tuning so the verified run is one application."""
        w, ttb = self.w, self.ttb
        if w.beta != 0.0:
            ttb.fill_uniform(w.kind, self.b_ext, None, w.seed_b, self.b.data_ptr(),
                             origin=self.b_org, global_sizes=w.sizes_b)

    def run(self, stream=None):
        for plan, pa, pb, _, _, _ in self.plans:
            plan.execute(pa, pb, stream)

    def checksum(self):
        w, ttb = self.w, self.ttb
        total = 0
        sbpos = _strides(self.b_ext)
        for _, _, pb, q, origin, ext in self.plans:
            ext_b = [ext[self.sb_order[k]] for k in range(len(ext))]
            org_b = [origin[self.sb_order[k]] for k in range(len(ext))]
            total += ttb.checksum(w.kind, ext_b, self.b_ext, pb, origin=org_b,
                                  global_sizes=w.sizes_b)
        return total % (1 << 64)

    def free(self):
        self.a = self.b = None
        self.plans = []


def _prod(v):
    r = 1
    for x in v:
        r *= int(x)
    return r


def _strides(ext):
    out, acc = [], 1
    for e in ext:
        out.append(acc)
        acc *= int(e)
    return out


def variant_of(plan_text):
    """Kernel that runs a plan: the `fn` key of ttb_plan_describe."""
    kv = dict(p.split("=", 1) for p in plan_text.split(";") if "=" in p)
    fn = kv.get("fn", kv.get("kern", "?"))
    return "btile" if fn == "btile_lin" else fn  # one kernel, two consumer walks


# ------------------------------------------------------------ reference arm --

def reference_rows(slab_div: int, max_rows=None):
    """Bounded sample of the sweep for the CPU: from every row the leading slab
    of B's outermost index (1/slab_div of it, at least one index), i.e. the
    same access pattern as the full row over fewer outer iterations."""
    rows = []
    for w in _workloads().C5[:max_rows]:
        outer_axis = w.gather[-1]
        ext = list(w.sizes)
        ext[outer_axis] = max(1, ext[outer_axis] // slab_div)
        rows.append((w, [0] * len(ext), ext))
    return rows


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


E2E_GROUP = 4         # host-buffer calls in flight at once in the e2e leg (4 x 2 x 1.6 GB pinned)
REF_SLAB_DIV = 16     # bounded sample: the leading 1/16 slab of every row
REF_TUNE_CAP = 8      # capped tune queue, prefetch distances {0, 5}


def time_reference(slab_div: int, steps: int, warmup: int, threads: int, max_rows=None):
    """The reference's best CPU path, per row: its B-linear nest
    (reference_transpose, executor.cpp:283-313) and execute_plan with the
    winner of its own tune over a capped queue (tuner.cpp:221-244 over
    build_candidates, search.cpp:243-303: max_implementations 8, prefetch
    distances {0, 5}), whichever is faster, on all host threads.  One code
    path for the --impl reference arm and the engine arm's cpu_baseline leg.
    Returns (GB/s, seconds per step, sample text)."""
    orc = _oracle()
    ref, co = orc.RefOracle(), orc.COracle()
    sessions = []
    n_plan = 0
    for w, origin, ext in reference_rows(slab_div, max_rows):
        s = orc.RefSession(ref, w.kind, w.kind, w.perm, ext, None, None, w.alpha, w.beta,
                           merge=True)
        A, B = s.a(), s.b()
        co.fill_uniform(w.kind, ext, None, w.seed_a, A)  # local data; timing is data-independent
        if w.beta != 0.0:
            sb = [0] * len(ext)
            for a, k in enumerate(w.perm):
                sb[k - 1] = ext[a]
            co.fill_uniform(w.kind, sb, None, w.seed_b, B)
        n = _prod(ext)
        nbytes = n * {"s": 4, "d": 8, "c": 8, "z": 16}[w.kind] * (3 if w.beta else 2)
        plan = None
        t_nest = min(s.run(threads) for _ in range(2))
        try:
            best, _ = s.tune(threads, max_impl=REF_TUNE_CAP, warmups=1, reps=3)
            t_plan = min(s.run(threads, best) for _ in range(2))
            if t_plan < t_nest:
                plan = best
                n_plan += 1
        except Exception:  # noqa: BLE001
            pass
        sessions.append((s, plan, nbytes))
    for _ in range(warmup):
        for s, plan, _ in sessions:
            s.run(threads, plan)
    # per row the minimum over the steps, as the reference's own timing
    # protocol takes the minimum of its repetitions (tuner.hpp:14-18)
    best = [float("inf")] * len(sessions)
    for _ in range(steps):
        for i, (s, plan, _) in enumerate(sessions):
            best[i] = min(best[i], s.run(threads, plan))
    total_bytes = sum(b for _, _, b in sessions)
    sec = sum(best)
    sample = (f"every c5 row, leading 1/{slab_div} slab of B's outermost index, "
              f"{len(sessions)} sub-problems, {total_bytes / 1e9:.2f} GB/step; per row the faster of "
              f"reference_transpose and execute_plan(tune cap {REF_TUNE_CAP}, d in {{0,5}}) "
              f"({n_plan} rows took the tuned plan); per row the best of {steps} steps")
    for s, _, _ in sessions:
        s.close()
    return total_bytes / 1e9 / sec, sec, sample


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    try:
        if not _oracle().have_ref():
            raise FileNotFoundError("oracle/_ref/libttune_ref.so not built")
        gbs, sec, sample = time_reference(REF_SLAB_DIV, args.steps, args.warmup, threads)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}))
        return 0
    line = {
        "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic (seeded counter-based generator, SURVEY s8(d))",
        "config": config_block(args.gpus), "impl": "reference",
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads,
                         "kind": "reference", "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------- engine arm --

def measure_d2d(torch):
    n = 1 << 28  # 1 GiB of fp32
    a = torch.empty(n, dtype=torch.float32, device="cuda")
    b = torch.empty_like(a)
    a.fill_(1.0)
    for _ in range(3):
        b.copy_(a)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e30
    for _ in range(5):
        e0.record()
        b.copy_(a)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * n * 4 / 1e9 / (best / 1e3)


def bench_configs(torch, ttb, peak, d2d):
    """c1-c4s at full size on one GPU: autotuned plan, best of 10 after 5 warm-ups (the
    reference takes minima of repetitions too, tuner.hpp:14-18; 70-300 us kernels)."""
    from paper_1603_02297_b200.workloads import CONFIGS
    golden = golden_checksums()
    out = {}
    for w in CONFIGS:
        p = ttb.make_problem(w.perm, list(w.sizes), w.kind, w.kind, w.alpha, w.beta,
                             w.lda and list(w.lda), w.ldb and list(w.ldb))
        na, nb = ttb.required_elements_a(p), ttb.required_elements_b(p)
        a, b = ttb.TensorBuffer(w.kind, na), ttb.TensorBuffer(w.kind, nb)
        ttb.fill_sentinel(w.kind, na, a.data_ptr())
        ttb.fill_uniform(w.kind, list(w.sizes), w.lda and list(w.lda), w.seed_a, a.data_ptr())
        plan = ttb.GpuPlan(p)
        plan.autotune(a, b, warmups=2, reps=6)
        if w.beta != 0.0:
            ttb.fill_uniform(w.kind, w.sizes_b, w.ldb and list(w.ldb), w.seed_b, b.data_ptr())
        plan.execute(a, b)
        ok = ttb.checksum(w.kind, w.sizes_b, w.ldb and list(w.ldb), b.data_ptr()) == golden[w.name]
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        for _ in range(5):
            plan.execute(a, b)
        best = 1e30
        for _ in range(10):
            e0.record()
            plan.execute(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        gbs = w.algorithmic_bytes / 1e9 / (best / 1e3)
        # a device-to-device copy of the same logical bytes, timed the same way:
        # what ramp and tail cost a 70-300 us kernel (beta != 0 reads B as well,
        # so its copy moves 3/2 of the tensor bytes: n elements in, n out, n/2 extra)
        nel = max(1, w.algorithmic_bytes // 8)
        src = torch.empty(nel, dtype=torch.float32, device="cuda")
        dst = torch.empty_like(src)
        for _ in range(5):
            dst.copy_(src)
        cbest = 1e30
        for _ in range(10):
            e0.record()
            dst.copy_(src)
            e1.record()
            e1.synchronize()
            cbest = min(cbest, e0.elapsed_time(e1))
        same = 2 * nel * 4 / 1e9 / (cbest / 1e3)
        del src, dst
        out[w.name] = {"gbs": round(gbs, 1), "pct_hbm": round(100 * gbs / peak, 1),
                       "pct_d2d": round(100 * gbs / d2d, 1), "us": round(best * 1e3, 1),
                       "d2d_same_bytes_gbs": round(same, 1),
                       "pct_d2d_same_bytes": round(100 * gbs / same, 1),
                       "plan": plan.describe(), "checksum_ok": ok}
        del a, b, plan
        torch.cuda.empty_cache()
    vals = [v["gbs"] for v in out.values()]
    same = [v["pct_d2d_same_bytes"] for v in out.values()]
    out["mean_gbs"] = round(sum(vals) / len(vals), 1)
    out["mean_pct_d2d"] = round(100 * out["mean_gbs"] / d2d, 1)
    out["mean_pct_d2d_same_bytes"] = round(sum(same) / len(same), 1)
    return out


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return {}


def run_engine_arm(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    ndev = torch.cuda.device_count()
    # NCCL over NVLink when every rank has its own GPU; gloo (host) when ranks
    # share a device (logic checks only -- the data path never communicates)
    backend = "nccl" if ndev >= world else "gloo"
    if world > 1:
        torch.cuda.set_device(local % ndev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(0)
    import paper_1603_02297_b200 as ttb
    from paper_1603_02297_b200.workloads import C5

    peak, peak_kind = peaks()
    golden = golden_checksums()
    coll_dev = "cuda" if backend == "nccl" else "cpu"

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t_setup = time.time()
    d2d = measure_d2d(torch)
    rows = [Row(w, world, rank, torch, ttb) for w in C5]
    for r in rows:
        r.allocate()
    for r in rows:
        r.autotune()
        r.refill_b()
    torch.cuda.synchronize()
    # verification run: one application per row, checksums gathered over NCCL
    for r in rows:
        r.run()
    sums = [r.checksum() for r in rows]
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, sums)
    else:
        gathered = [sums]
    checks_ok = all(sum(g[i] for g in gathered) % (1 << 64) == golden[w.name]
                    for i, w in enumerate(C5))
    log(f"[rank {rank}] setup+tune+verify {time.time() - t_setup:.1f}s, checksums ok={checks_ok}")

    stream = torch.cuda.current_stream()
    # A step issues the rows back to back on one stream (`--streams 1`, the
    # default).  The rows are independent problems, so `--streams N` can issue
    # them round-robin on N streams; measured on B200 it changes nothing (6057
    # vs 6058 GB/s: the sweep runs at the power cap, not at kernel boundaries).
    # The step is bracketed on the main stream: side streams wait for e_start
    # and the main stream for every side stream before e_stop.
    nstreams = max(1, args.streams)
    side = [stream] + [torch.cuda.Stream() for _ in range(nstreams - 1)]
    joins = [torch.cuda.Event() for _ in side]

    def step(e0, e1):
        e0.record(stream)
        for st in side[1:]:
            st.wait_event(e0)
        for i, r in enumerate(rows):
            r.run(side[i % nstreams])
        for st, j in zip(side[1:], joins[1:]):
            j.record(st)
            stream.wait_event(j)
        e1.record(stream)

    e_start, e_stop = torch.cuda.Event(True), torch.cuda.Event(True)
    for _ in range(args.warmup):
        step(e_start, e_stop)
    # a second pass of the same steps with an event pair per row on the
    # launching stream (kernel share, per-row rates, roofline); the pairs cost
    # ~1.5% of the step, so `value` comes from the plain pass above
    ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in rows]
    row_ms = [0.0] * len(rows)
    step_ms, serial_ms = [], []
    launches0 = ttb.launch_count()
    with ClockSampler(local % ndev) as clk:
        barrier()
        torch.cuda.nvtx.range_push("ttb_timed")  # ncu --nvtx-include "ttb_timed/"
        for _ in range(args.steps):
            step(e_start, e_stop)
            e_stop.synchronize()
            step_ms.append(e_start.elapsed_time(e_stop))
        torch.cuda.nvtx.range_pop()
        launches = ttb.launch_count() - launches0
        barrier()
        for _ in range(args.steps):
            e_start.record(stream)
            for i, r in enumerate(rows):
                ev[i][0].record(stream)
                r.run(stream)
                ev[i][1].record(stream)
            e_stop.record(stream)
            e_stop.synchronize()
            serial_ms.append(e_start.elapsed_time(e_stop))
            for i in range(len(rows)):
                row_ms[i] += ev[i][0].elapsed_time(ev[i][1])
        barrier()
    local_ms = sum(step_ms) / len(step_ms)
    local_serial_ms = sum(serial_ms) / len(serial_ms)
    ms = allmax(local_ms)
    total_bytes = sum(w.algorithmic_bytes for w in C5)
    value = total_bytes / 1e9 / (ms / 1e3)

    # dominant kernel family and its roofline (algorithmic bytes / launch time)
    fam_ms, fam_bytes, fam_launch = {}, {}, {}
    per_row = []
    for i, r in enumerate(rows):
        fam = variant_of(r.plans[0][0].describe()) if r.plans else "none"
        t = row_ms[i] / args.steps
        fam_ms[fam] = fam_ms.get(fam, 0.0) + t
        fam_bytes[fam] = fam_bytes.get(fam, 0) + r.bytes
        fam_launch[fam] = fam_launch.get(fam, 0) + len(r.plans)
        per_row.append({"row": r.w.name, "gbs": round(r.bytes / 1e9 / (t / 1e3), 1),
                        "plan": r.plans[0][0].describe() if r.plans else None})
    dom = max(fam_ms, key=fam_ms.get)
    achieved = fam_bytes[dom] / 1e9 / (fam_ms[dom] / 1e3)
    traffic = load_traffic().get(dom)
    roofline = {"bound": "hbm", "kernel": f"{dom}_kernel", "achieved": round(achieved, 1),
                "peak": peak, "peak_source": peak_kind, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "share_of_step": round(fam_ms[dom] / local_serial_ms, 3),
                "algorithmic_bytes_per_launch": fam_bytes[dom] // max(fam_launch[dom], 1)}

    for r in rows:
        r.free()
    torch.cuda.empty_cache()
    # end-to-end through the public API with pinned host buffers
    e2e = None if args.no_e2e else run_e2e(torch, ttb, rows, world, allmax, steps=min(args.steps, 3))

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic (seeded counter-based generator, SURVEY s8(d))",
        "config": config_block(world), "streams": nstreams, "roofline": roofline, "e2e": e2e,
        "clocks": clk.summary(), "gpu_launches": launches,
        "pct_hbm_peak": round(100 * value / (peak * world), 2),
        "d2d_memcpy_gbs": round(d2d, 1), "pct_d2d": round(100 * value / (d2d * world), 2),
        "checksums_ok": checks_ok, "rows": per_row,
        "per_row_pass": {"ms_per_step": round(allmax(local_serial_ms), 4),
                         "value": round(total_bytes / 1e9 / (allmax(local_serial_ms) / 1e3), 2),
                         "note": "the same steps again with an event pair per row (one stream): "
                                 "the pass `rows` and `roofline` are timed in"},
    }
    torch.cuda.empty_cache()
    if rank == 0 and world == 1:
        if not args.no_configs:
            line["configs"] = bench_configs(torch, ttb, peak, d2d)
        if not args.no_cpu:
            # the reference arm itself, in a fresh process: inside this one (CUDA
            # context, pinned allocations, torch's thread pools) the same
            # function measured up to 25% lower than the arm run on its own
            try:
                env = {k: v for k, v in os.environ.items()
                       if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE")}
                r = subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "reference",
                                    "--steps", "5", "--warmup", "3"], env=env, capture_output=True,
                                   text=True, timeout=900)
                ref_line = json.loads(r.stdout.strip().splitlines()[-1])
                if "unavailable" in ref_line:
                    raise RuntimeError(ref_line["unavailable"])
                line["cpu_baseline"] = ref_line["cpu_baseline"]
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "unit": "GB/s", "cores": 0,
                                        "kind": "reference", "sample": f"failed: {e}"}
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def measure_pcie(torch, nbytes=1 << 30):
    """Pinned host <-> device copy bandwidth (GB/s): H2D alone, D2H alone, and
    both at once on two streams (PCIe is full duplex) -- the e2e roofline."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=3):
        best = 1e30
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    t_h2d = timed(lambda: d.copy_(h, non_blocking=True))
    t_d2h = timed(lambda: h2.copy_(d2, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    t_both = timed(both)
    del h, h2, d, d2
    torch.cuda.empty_cache()
    return {"h2d_gbs": round(nbytes / 1e9 / t_h2d, 1), "d2h_gbs": round(nbytes / 1e9 / t_d2h, 1),
            "both_gbs": round(2 * nbytes / 1e9 / t_both, 1)}


def run_e2e(torch, ttb, rows, world, allmax, steps):
    """Same metric through GpuPlan.execute_host: per row, H2D of the inputs from
    pinned host memory, the kernel, D2H of B, all inside the timed region."""
    import numpy as np
    plans = []
    max_a = max_b = 0
    for r in rows:
        for origin, ext in r.boxes:
            w = r.w
            q = ttb.make_problem(w.perm, ext, w.kind, w.kind, w.alpha, w.beta)
            na = ttb.required_elements_a(q) * r.kind.components
            nb = ttb.required_elements_b(q) * r.kind.components
            plans.append((r, q, ttb.GpuPlan(q), origin, ext, na, nb))
            sz = 8 if w.kind in "dz" else 4
            max_a, max_b = max(max_a, na * sz), max(max_b, nb * sz)
    # E2E_GROUP transpositions are in flight at once (execute_host(wait=False),
    # then host_sync each): the next one's host->device copies run while the
    # previous one's last slabs compute and stream out.  Each in-flight call
    # has its own pinned buffer pair; the inputs are set up untimed per group.
    G = max(1, min(E2E_GROUP, len(plans)))
    host_a = [torch.empty(max_a, dtype=torch.uint8, pin_memory=True) for _ in range(G)]
    host_b = [torch.empty(max_b, dtype=torch.uint8, pin_memory=True) for _ in range(G)]
    h2d = d2h = 0
    total = 0.0
    for step in range(steps):
        for g0 in range(0, len(plans), G):
            group = plans[g0:g0 + G]
            bufs = []
            for slot, (r, q, plan, origin, ext, na, nb) in enumerate(group):
                w = r.w
                dt = np.float64 if w.kind in "dz" else np.float32
                sz = 8 if w.kind in "dz" else 4
                ha = host_a[slot][: na * sz].numpy().view(dt)
                hb = host_b[slot][: nb * sz].numpy().view(dt)
                # setup (untimed): this box's inputs from the device generator
                dev = torch.empty(max(na, nb), dtype=torch.float64 if sz == 8 else torch.float32,
                                  device="cuda")
                ttb.fill_uniform(w.kind, ext, None, w.seed_a, dev.data_ptr(), origin=origin,
                                 global_sizes=list(w.sizes))
                torch.cuda.synchronize()
                ha[:] = dev[:na].cpu().numpy()
                if w.beta != 0.0:
                    sbx = ttb.sizes_b(q)
                    org_b = [origin[a] for a in sorted(range(len(ext)), key=lambda a: w.perm[a])]
                    ttb.fill_uniform(w.kind, sbx, None, w.seed_b, dev.data_ptr(), origin=org_b,
                                     global_sizes=w.sizes_b)
                    torch.cuda.synchronize()
                    hb[:] = dev[:nb].cpu().numpy()
                del dev
                if step == 0:
                    plan.execute_host(ha, hb)  # first call allocates the plan's staging
                    h2d += na * sz + (nb * sz if w.beta != 0.0 else 0)
                    d2h += nb * sz
                bufs.append((plan, ha, hb))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for plan, ha, hb in bufs:
                plan.execute_host(ha, hb, wait=False)
            for plan, ha, hb in bufs:
                plan.host_sync()
            total += time.perf_counter() - t0
    per_step = allmax(total / steps)
    nbytes = sum(w.algorithmic_bytes for w in {id(r.w): r.w for r in rows}.values())
    del host_a, host_b
    torch.cuda.empty_cache()
    # PCIe roofline: no schedule can beat either direction alone at its own
    # rate, nor all the bytes at the measured duplex rate
    pcie = measure_pcie(torch)
    t_min = max(h2d / 1e9 / pcie["h2d_gbs"], d2h / 1e9 / pcie["d2h_gbs"],
                (h2d + d2h) / 1e9 / pcie["both_gbs"])
    roof = nbytes / 1e9 / t_min if t_min > 0 else None
    value = nbytes / 1e9 / per_step
    return {"value": round(value, 3), "unit": "GB/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(per_step * 1e3, 2), "steps": steps,
            "pcie": dict(pcie, roof_gbs=round(roof, 1) if roof else None,
                         frac=round(value / roof, 3) if roof else None),
            "in_flight": G,
            "path": "GpuPlan.execute_host(wait=False) + host_sync (ttb_plan_execute_host_async), "
                    "pinned host buffers, %d transpositions in flight" % G}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ttb", choices=["ttb", "reference"])
    ap.add_argument("--streams", type=int, default=1,
                    help="streams the independent rows of a step are issued on (1: back to back)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg (profiling runs)")
    ap.add_argument("--no-configs", action="store_true", help="skip the c1-c4s block (profiling runs)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        return spawn_ranks(args.gpus)
    if world is not None and int(world) != args.gpus:
        log(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
        return 2
    if args.gpus > 1:
        # the communicator's init lines (nranks) in the log of every rank
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_engine_arm(args)


def spawn_ranks(n: int) -> int:
    """`--gpus N` outside torchrun: start N ranks of this command on this node
    (the torchrun environment: RANK / LOCAL_RANK / WORLD_SIZE / MASTER_*),
    rank 0's stdout carries the JSON line; exit code = worst rank's."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, *sys.argv], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


if __name__ == "__main__":
    sys.exit(main())
