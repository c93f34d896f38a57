"""msGeMM benchmark (driver contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

Workload (default): BASELINE.json config 5 -- W 65536x8192 int4, X 8192x8
fp16 ~N(0,1), d=3 -- the configuration the metric's "1/2/4/8 B200" refers to
and the largest single-GPU one.  At N GPUs the 65536 rows are sharded over
the ranks (strong scaling: total work fixed) and the Y slices are
all-gathered with NCCL.  A "step" is one full msGeMM of the config.

Metric: effective GOP/s = 2*m*k*b / step time (whole job), plus the HBM
roofline of the dominant kernel (fused LUT kernel) and end-to-end numbers
through the public API with pinned host buffers.  L2 reuse across steps is
defeated by rotating over >= 3x L2 worth of distinct weight copies.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2310_06178_b200.workloads import CONFIGS, algorithmic_bytes, effective_ops  # noqa: E402

L2_BYTES = 126 * 1024 * 1024
EXTRA_FLAGS = int(os.environ.get("MSG_BENCH_FLAGS", "0"))  # experiments only (C-ABI flag bits)
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)",
                "sm_max_mhz": d.get("sm_max_mhz")}
    return dict(PEAKS_FALLBACK)


# --------------------------------------------------------------------------- clocks
_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
            0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
            0x100: "display_clock_setting"}


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons via NVML while the timed region runs."""

    def __init__(self, torch_dev):
        super().__init__(daemon=True)
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._halt = threading.Event()
        self.ok = False
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(torch_dev).uuid)
            uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
            self.h = pynvml.nvmlDeviceGetHandleByUUID(uuid.encode())
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - reported in the JSON
            self.err = repr(e)

    def sample(self):
        if not self.ok:
            return
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for bit, name in _REASONS.items():
            if mask & bit:
                self.reasons.add(name)

    def run(self):
        while not self._halt.is_set():
            self.sample()
            time.sleep(0.005)

    def stop(self):
        self._halt.set()
        self.join(timeout=1)
        self.sample()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons - {"gpu_idle"})}


# --------------------------------------------------------------------------- CPU baseline
class CpuArm:
    """The oracle port (numpy restatement of the reference's msgemm) on the same
    workload, host threads across batch columns (the reference's own
    ThreadPool split, gemm.py:136-152; workers=1 is the reference as shipped)."""

    def __init__(self, cfg):
        from oracle import msgemm_oracle as orc
        from paper_2310_06178_b200.workloads import activations, weights
        self.orc, self.cfg = orc, cfg
        self.data = weights(cfg)
        X = activations(cfg)
        self.X = X.astype(np.int64) if cfg.x_dtype == "int" else X
        self.host_cores = len(os.sched_getaffinity(0))
        self.cores = min(self.host_cores, max(cfg.b, 1))
        self.vals = orc.int4_values()

    def run(self, r0, rows, workers=None):
        cfg = self.cfg
        r0 = r0 % max(cfg.m - rows + 1, 1)
        t0 = time.perf_counter()
        self.orc.msgemm(self.data[r0:r0 + rows], rows, cfg.k, 4, self.vals, self.X, cfg.d,
                        workers=self.cores if workers is None else workers)
        return time.perf_counter() - t0

    def fit(self, workers):
        """Per-call cost t(rows) = a + c * rows (a: the per-column table builds,
        c: gathers + row sums), from two sample sizes."""
        r1, r2 = min(self.cfg.m, 512), min(self.cfg.m, 2048)
        t1, t2 = self.run(0, r1, workers), self.run(r1, r2, workers)
        c = max((t2 - t1) / max(r2 - r1, 1), 1e-9)
        return max(t1 - c * r1, 0.0), c

    def gops(self, rows, seconds):
        return 2.0 * rows * self.cfg.k * self.cfg.b / seconds / 1e9

    def describe(self, rows, seconds, nsteps=1, workers=None):
        cfg = self.cfg
        what = "the full workload" if rows == cfg.m else f"{rows} rows of {cfg.m}"
        return (f"oracle port (numpy, reference algorithm) on {nsteps} x {what} "
                f"(k={cfg.k}, b={cfg.b}, d={cfg.d}), workers={self.cores if workers is None else workers}, "
                f"{seconds:.2f}s total")


def cpu_baseline(cfg, budget_s: float = 30.0):
    """Both variants of SURVEY.md 8(d): workers=N threads across columns (the
    reported value: the full workload when it fits the budget) and workers=1
    as shipped (a row sample, extrapolated to the full workload with the
    fitted per-call cost)."""
    arm = CpuArm(cfg)
    variants = []
    for workers in (arm.cores, 1):
        a, c = arm.fit(workers)
        full_est = a + c * cfg.m
        share = budget_s * (0.6 if workers > 1 else 0.3)
        rows = cfg.m if full_est <= share else int(min(cfg.m, max(64, (share - a) / c)))
        t = arm.run(0, rows, workers)
        v = {"workers": workers, "value": arm.gops(rows, t), "unit": "GOP/s",
             "sample": arm.describe(rows, t, 1, workers),
             "full_workload": rows == cfg.m}
        if rows != cfg.m:
            v["extrapolated_full_value"] = arm.gops(cfg.m, a + c * cfg.m)
            v["fit_s"] = {"per_call": a, "per_row": c}
        variants.append(v)
    main = variants[0]
    return {"value": main["value"], "unit": "GOP/s", "cores": arm.cores, "kind": "port",
            "sample": main["sample"], "same_config": main["full_workload"],
            "host_cores": arm.host_cores, "variants": variants}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (oracle port) on this host
    with all the threads it can use, each step a bounded row sample (the whole
    run stays within a few minutes).  The per-call cost fit extrapolates the
    sample to the full workload (reported beside the measured value)."""
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    arm = CpuArm(cfg)
    a, c = arm.fit(arm.cores)
    per_step = min(5.0, max(0.05, 120.0 / max(args.steps + args.warmup, 1)))
    rows = cfg.m if a + c * cfg.m <= per_step else int(min(cfg.m, max(16, (per_step - a) / c)))
    for i in range(args.warmup):
        arm.run(i * rows, rows)
    total = 0.0
    for i in range(args.steps):
        total += arm.run((args.warmup + i) * rows, rows)
    value = arm.gops(rows * args.steps, total)
    out = {
        "metric": "effective GOP/s (2*m*k*b/time) and achieved HBM GB/s vs roofline",
        "value": value, "unit": "GOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f16" if cfg.x_dtype == "float16"
        else cfg.x_dtype, "data": "synthetic (seeded numpy default_rng)", "impl": "reference",
        "config": {"workload": cfg.name, "m": cfg.m, "k": cfg.k, "b": cfg.b, "d": cfg.d,
                   "step": "the full workload" if rows == cfg.m else
                           f"{rows}-row sample of the workload"},
        "cpu_baseline": {"value": value, "unit": "GOP/s", "cores": arm.cores, "kind": "port",
                         "sample": arm.describe(rows, total, args.steps)},
        "e2e": {"value": value, "unit": "GOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if rows != cfg.m:
        out["cpu_baseline"].update(extrapolated_full_value=arm.gops(cfg.m, a + c * cfg.m),
                                   fit_s={"per_call": a, "per_row": c})
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="cfg5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--gather", default="nccl", choices=["nccl", "peer"],
                    help="row shards: NCCL all-gather of the Y slices (default), or the all-gather "
                         "fused into the finishing kernels over symmetric memory (peer stores; "
                         "opt-in: this pool has no multi-GPU box to measure it on)")
    ap.add_argument("--split", default="rows", choices=["rows", "k"],
                    help="N>1: shard rows (+ all-gather of Y, default) or the inner dimension "
                         "(+ fp32 all-reduce of partial Y; splits the table build too)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2310_06178_b200 as mg
    from paper_2310_06178_b200 import _lib
    from paper_2310_06178_b200.workloads import activations, weights

    # functional test of the N > 1 code path on a one-GPU box only
    # (tests/test_bench_multirank.py): every rank on cuda:0, gloo collectives.
    # Never a measurement: ranks sharing a GPU are not N GPUs.
    share = os.environ.get("MSG_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    ksplit = world > 1 and args.split == "k"
    X = activations(cfg)
    exact = cfg.x_dtype == "int"
    Xh = X.astype(np.float16) if exact else X
    kw = dict(table_dtype=np.float32, out_dtype=np.float32) if exact else {}
    if ksplit:
        # rank owns columns [k0, k1) of every row; partial Y in fp32, summed by NCCL
        from paper_2310_06178_b200.sharded import k_split_bounds
        k0, k1 = k_split_bounds(cfg.k, cfg.d, world, rank)
        mr, kr = cfg.m, k1 - k0
        data = np.ascontiguousarray(weights(cfg)[:, k0 // 2:(k1 + 1) // 2])
        xd = torch.from_numpy(np.ascontiguousarray(Xh[k0:k1])).to(dev)
        kw = dict(kw, out_dtype=np.float32)
        y_dt = torch.float32
    else:
        if cfg.m % world:
            raise SystemExit(f"m={cfg.m} not divisible by {world} ranks")
        mr, kr = cfg.m // world, cfg.k
        r0 = rank * mr
        k0, k1 = 0, cfg.k
        data = weights(cfg)[r0:r0 + mr]
        xd = torch.from_numpy(Xh).to(dev)
        y_dt = torch.float32 if exact else xd.dtype

    # distinct weight copies so consecutive steps never hit in L2
    shard_bytes = data.nbytes
    ncopies = max(2, math.ceil(3 * L2_BYTES / shard_bytes))
    base = torch.from_numpy(data).to(dev)
    pwms = []
    for c in range(ncopies):
        dd = base if c == 0 else base.clone()
        pwms.append(mg.PackedWeightMatrix(m=mr, k=kr, width=4, data=dd,
                                          codebook=mg.int4_codebook()))
    Yshard = torch.empty((mr, cfg.b), dtype=y_dt, device=dev)
    Yfull = torch.empty((cfg.m, cfg.b), dtype=y_dt, device=dev) if world > 1 else Yshard
    peer_y = None
    if world > 1 and not ksplit and not share and args.gather == "peer":
        from paper_2310_06178_b200.sharded import PeerY
        peer_y = PeerY(cfg.m, cfg.b, y_dt, dev)       # Y in symmetric memory on every rank
        Yfull, Yshard = peer_y.buf, peer_y.local()
        os.environ["MSG_BENCH_NO_GRAPH"] = "1"        # the signal-pad barrier is not captured

    def collective():
        if peer_y is not None:   # the finishing kernels already stored into every rank's Y
            peer_y.barrier()
            return
        if share:      # gloo functional test: host-staged collectives
            if ksplit:
                h = Yshard.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.SUM)
                Yshard.copy_(h)
            else:
                h = torch.empty((cfg.m, cfg.b), dtype=Yshard.dtype)
                dist.all_gather_into_tensor(h, Yshard.cpu())
                Yfull.copy_(h)
        elif ksplit:
            dist.all_reduce(Yshard, op=dist.ReduceOp.SUM)   # Yshard: this rank's fp32 partial
        else:
            dist.all_gather_into_tensor(Yfull, Yshard)
    TC = -1  # pseudo-flag: the dense dequantise-then-multiply comparison kernel (K4) instead of msGeMM
    xd16 = xd.half()
    Ytc = torch.empty((mr, cfg.b), dtype=torch.float32, device=dev)

    def step(i, flags=0, gather=True):
        if flags == TC:
            mg.dequant_gemm(pwms[i % ncopies], xd16, out=Ytc)
            return
        fan = peer_y.targets() if (peer_y is not None and not flags and gather) else None
        mg.msgemm(pwms[i % ncopies], xd, cfg.d, out=Yshard, _flags=flags | EXTRA_FLAGS, _fan=fan, **kw)
        if world > 1 and not flags and gather:
            collective()

    def barrier():
        if world > 1:
            dist.barrier()

    use_graphs = os.environ.get("MSG_BENCH_NO_GRAPH", "0") != "1"
    graphs = {}

    def graph_for(n, flags, start=0):
        """One CUDA graph holding the kernels of n consecutive steps (weight copies
        start..start+n-1 mod ncopies): launches replay without host overhead.
        Collectives are never captured; with N > 1 ranks each step replays a
        one-step graph and then all-gathers eagerly."""
        key = (n, flags, start)
        if key not in graphs:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(start, start + n):
                    step(i, flags, gather=False)
            graphs[key] = g
        return graphs[key]

    def timed(nsteps, flags=0):
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if use_graphs and world == 1:
            per = ncopies * max(1, math.ceil(8 / ncopies))
            reps, rem = divmod(nsteps, per)
            g_full = graph_for(per, flags) if reps else None
            g_rem = graph_for(rem, flags) if rem else None
            e0.record()
            for _ in range(reps):
                g_full.replay()
            if rem:
                g_rem.replay()
            e1.record()
        elif use_graphs:
            gs = [graph_for(1, flags, c) for c in range(ncopies)]
            e0.record()
            for i in range(nsteps):
                gs[i % ncopies].replay()
                if flags == 0:
                    collective()
            e1.record()
        else:
            e0.record()
            for i in range(nsteps):
                step(i, flags)
            e1.record()
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ms], device="cpu" if share else dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = tt.item()
        return ms / nsteps

    for i in range(max(args.warmup, ncopies)):     # also builds every copy's repacked layout
        step(i)
    torch.cuda.synchronize()

    timed(min(args.steps, 16))                        # capture + warm the graphs
    sampler = ClockSampler(dev)
    sampler.start()
    ms_step = timed(args.steps)
    sampler.stop()
    clocks = sampler.summary()

    # dominant kernel alone (fused LUT kernel; finish kernel and all-gather skipped)
    for i in range(3):
        step(i, _lib.FLAG_LUT_PHASE_ONLY)
    timed(min(args.steps, 16), _lib.FLAG_LUT_PHASE_ONLY)
    ms_lut = timed(args.steps, _lib.FLAG_LUT_PHASE_ONLY)
    torch.cuda.synchronize()
    _lib.reset_workspaces()   # LUT-only launches of the b=1 kernel leave their sums behind
    # the dense tensor-core baseline on the same shard (context, not the metric)
    ms_tc = None
    if cfg.b <= 256:
        for i in range(max(3, ncopies)):
            step(i, TC)
        timed(min(args.steps, 16), TC)
        ms_tc = timed(args.steps, TC)

    # end to end through the public API: pinned host X in, host Y out, every step
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 50))
    Xpin = torch.from_numpy(Xh).pin_memory()
    Ypin = torch.empty((cfg.m, cfg.b), dtype=y_dt, pin_memory=True)

    def e2e_step(i):
        if world == 1:
            mg.msgemm(pwms[i % ncopies], Xpin, cfg.d, out=Ypin, **kw)
        elif ksplit:
            x_dev = Xpin[k0:k1].to(dev, non_blocking=True)
            mg.msgemm(pwms[i % ncopies], x_dev, cfg.d, out=Yshard, **kw)
            collective()
            Ypin.copy_(Yshard.to(Ypin.dtype))
        else:
            x_dev = Xpin.to(dev, non_blocking=True)
            mg.msgemm(pwms[i % ncopies], x_dev, cfg.d, out=Yshard, **kw)
            collective()
            Ypin.copy_(Yfull)

    for i in range(2 * ncopies + 1):    # each copy's host-path graph is captured on its 2nd call
        e2e_step(i)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        e2e_step(i)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = 1e3 * (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        tt = torch.tensor([e2e_ms], device="cpu" if share else dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = tt.item()

    # which LUT kernel the plan runs, and K3 (the one-time weight repack) timed alone
    plan = next(v for kk, v in pwms[0]._device_cache.items() if kk[0] == "call")
    kernel_name = {_lib.LAYOUT_LANE: "lane_lut_kernel", _lib.LAYOUT_RB4: "rb_tmem_kernel<16>",
                   _lib.LAYOUT_RB4S: "rb_tmem_kernel<8>",
                   _lib.LAYOUT_RB8: "rb_lut_kernel<4>", _lib.LAYOUT_RB16: "rb_lut_kernel<2>",
                   _lib.LAYOUT_QUAD: "fused_lut_kernel"}.get(plan.layout, "generic_gemm_kernel")
    k3 = None
    if plan.layout != _lib.LAYOUT_NONE:
        lib = _lib.lib()
        rep_bytes = int(lib.msg_repacked_bytes(mr, kr, cfg.d, plan.layout))
        scratch = torch.empty(rep_bytes, dtype=torch.uint8, device=dev)
        sp = torch.cuda.current_stream().cuda_stream

        def repack(i):
            _lib.check(lib.msg_repack(_lib.ptr(pwms[i % ncopies].data), mr, kr, cfg.d, plan.layout,
                                      plan.symmetric, _lib.ptr(scratch), sp))
        for i in range(2):
            repack(i)
        torch.cuda.synchronize()
        nrep = 6
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(nrep):
            repack(i)
        e1.record()
        torch.cuda.synchronize()
        ms_k3 = e0.elapsed_time(e1) / nrep
        k3_bytes = shard_bytes + rep_bytes
        del scratch
        k3 = {"kernel": "K3 repack (" + {_lib.LAYOUT_LANE: "lane", _lib.LAYOUT_RB4: "rb4",
                                           _lib.LAYOUT_RB4S: "rb4s",
                                           _lib.LAYOUT_RB8: "rb8", _lib.LAYOUT_RB16: "rb16",
                                           _lib.LAYOUT_QUAD: "quad"}[plan.layout] + " layout)",
              "ms": ms_k3, "bytes": k3_bytes, "gbs": k3_bytes / (ms_k3 * 1e-3) / 1e9,
              "frac": k3_bytes / (ms_k3 * 1e-3) / 1e9 / load_peaks()["hbm_gbs"],
              "note": "one-time per weight matrix, excluded from the step"}

    ops = effective_ops(cfg)
    value = ops / (ms_step * 1e-3) / 1e9
    peaks = load_peaks()
    shard_cfg = type(cfg)(cfg.name, mr, kr, cfg.b, cfg.d, cfg.x_dtype, cfg.seed)
    x_item = Xh.dtype.itemsize                      # fp16 (or fp32 for config 1)
    f32_tables = exact or x_item == 4
    y_item = 4 if f32_tables else 2
    lane = plan.layout == _lib.LAYOUT_LANE
    bytes_launch = algorithmic_bytes(shard_cfg, x_itemsize=x_item, y_itemsize=y_item)
    achieved = bytes_launch / (ms_lut * 1e-3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get(f"{cfg.name}@{world}")
    nb = kr // cfg.d
    e_item = 4 if f32_tables else 2
    smem_bytes = (mr * nb + 2048 * nb) * cfg.b * e_item     # LUT reads + half-table writes
    out = {
        "metric": "effective GOP/s (2*m*k*b/time) and achieved HBM GB/s vs roofline",
        "value": value, "unit": "GOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if x_item == 4 else "f16",
        "data": "synthetic (seeded numpy default_rng; uniform int4 W, "
                + ("integer X in [-127, 127]" if exact else "N(0,1) X") + ")",
        "config": {"workload": cfg.name, "m": cfg.m, "k": cfg.k, "b": cfg.b, "d": cfg.d,
                   "x": "fp32" if x_item == 4 else "fp16",
                   "tables": ("fp32 sign-symmetric half tables" if f32_tables else
                              "fp16 sign-symmetric half tables (2048/group"
                              + (", 32 bank-private per chunk)" if lane else ")")),
                   "accum": "int64 fixed point across CTAs" if lane else "f32",
                   "y": "fp32" if f32_tables else "fp16",
                   "parallelism": (f"row-shard x{world} + all-gather fused into the finishing kernels "
                                   "(peer stores over symmetric memory)" if peer_y is not None else
                                   f"k-split x{world} + NCCL fp32 all-reduce" if ksplit else
                                   f"row-shard x{world}" + (" + NCCL all-gather" if world > 1 else "")),
                   "timing": "CUDA-graph replay of the K steps" if use_graphs else "eager launches",
                   "l2": f"rotate {ncopies} weight copies ({ncopies * shard_bytes / 2**20:.0f} MiB "
                         f">= 3x L2) between steps"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                     "kernel": kernel_name, "kernel_ms": ms_lut,
                     "kernel_share": ms_lut / ms_step, "algorithmic_bytes_per_launch": bytes_launch,
                     "peak_source": peaks["source"],
                     "smem_lut_bytes_per_launch": smem_bytes,
                     "smem_lut_tbs": smem_bytes / (ms_lut * 1e-3) / 1e12},
        "e2e": {"value": ops / (e2e_ms * 1e-3) / 1e9, "unit": "GOP/s",
                "ms_per_step": e2e_ms, "h2d_bytes_per_step": Xh[k0:k1].nbytes,
                "d2h_bytes_per_step": cfg.m * cfg.b * y_item,
                "path": "msgemm(pwm, pinned host X) -> host Y" if world == 1 else
                        ("H2D X slice, msgemm k-slice, NCCL all-reduce, D2H Y" if ksplit else
                         "H2D X, msgemm shard, NCCL all-gather, D2H Y")},
        "tensor_core_baseline": None if ms_tc is None else {
            "kernel": ("K4: weight-streaming int4->fp16 dequant + mma.sync m16n8k16, fp32 accumulation, "
                       "cluster split-k over DSMEM" if shard_cfg.b <= 16 and shard_cfg.k % 32 == 0 else
                       "K4: int4->fp16 dequant + tcgen05.mma kind::f16, fp32 TMEM accumulation"),
            "ms_per_step": ms_tc, "value": effective_ops(shard_cfg) / (ms_tc * 1e-3) / 1e9,
            "unit": "GOP/s (this rank's shard, no all-gather)",
            "hbm_frac": algorithmic_bytes(shard_cfg, 2, 4) / (ms_tc * 1e-3) / 1e9 / peaks["hbm_gbs"]},
        "k3_repack": k3,
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(cfg)
        out["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
