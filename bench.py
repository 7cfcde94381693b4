"""Benchmark: full W1+W2 (md + dp) kernelization on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl b200|reference]

A step is one complete kernelization to the fixpoint (reference
par_kernelize, parallel.py:164-214) of the config's synthetic instance.

* value     incidence-entries/s = n*m / (device time of one kernelization),
            instance resident in HBM (mhsk_kernelize_device), max over ranks.
* e2e       the same metric through the public C ABI with HOST buffers
            (mhsk_kernelize: pinned CSR -> device, alive flags -> host).
* roofline  dominant kernel = the tcgen05 Gram product: tensor ops per
            launch (the SYRK count M(M+1)K per phase, or the ops actually
            issued when exact pruning -- probe or block-sparse -- skipped
            MMAs; "pruned_ops_frac" = 1 - issued / algorithmic)
            / its CUDA-event time, against the dense peak of the operand
            format it ran on (FP4 kind::mxf4 for dense phases, int8 kind::i8
            for block-sparse ones).
* cpu_baseline / --impl reference: the reference's algorithm (oracle port,
            oracle/mhsk_oracle.c, all host threads) on a bounded sample of the
            same workload -- round-1 decisions for the first J items of each
            phase at full width K -- extrapolated to one full round.

Multi-GPU (torchrun, N>1): each rank runs a contiguous slice of every
phase's tile list; per-item deleter counts are summed with an NCCL
all-reduce between the Gram product and the commit (strong scaling).
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

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIG_DESC = {
    "c1": "random HS n=m=2000 p=0.05 alpha=1 (reference generate_random, seed)",
    "c2": "planted nested chains 100x100, alpha=3, 5% duplicate edges + twin vertices, n=m=10500",
    "c3": "stations x trains n=50000 m=20000 interval hyperedges, alpha=1",
    "c3a3": "stations x trains n=50000 m=20000 interval hyperedges, alpha=3",
    "c4": "random MHS n=m=100000 p=0.01 alpha=3 (counter-based generator)",
    "c5": "random MHS n=m=200000 p=0.01 alpha=5 (counter-based generator)",
}


def load_peaks() -> dict:
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML
    every 5 ms plus one sample on entry and one on exit (so even a
    millisecond-long region is covered); nvidia-smi polling if NVML is
    unavailable."""

    # nvmlClocksEventReason* bits
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}
    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.samples: list[tuple[float, float, int]] = []
        self.lines: list[str] = []
        self._stop = threading.Event()

    def _handle(self):
        import pynvml

        pynvml.nvmlInit()
        try:   # the CUDA device's NVML handle (indices differ under CUDA_VISIBLE_DEVICES)
            import torch

            props = torch.cuda.get_device_properties(self.index)
            pci = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(pci.encode())
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _sample(self):
        nv, h = self.nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        try:
            why = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except AttributeError:
            why = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.samples.append((float(sm), float(mx), int(why)))

    def _poll(self):
        while not self._stop.wait(0.005):
            self._sample()

    def __enter__(self):
        try:
            self.nvml = self._handle()
            self._sample()
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.nvml:
            try:
                self._sample()
            except Exception:
                pass
            self._stop.set()
            self._t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self._t.join(timeout=2)

    def summary(self) -> dict:
        sms, maxes, reasons = [], [], set()
        for sm, mx, why in self.samples:
            sms.append(sm)
            maxes.append(mx)
            reasons.update(name for name, bit in self.REASONS.items() if why & bit)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sms.append(float(parts[0]))
                maxes.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sms) if sms else None,
                "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(sms),
                "source": "nvml" if self.samples else "nvidia-smi"}


def make_instance(config: str, seed: int, ctx=None):
    """The config's instance.  Configs 4/5 (counter-based generator) are
    generated on the device when a context is given, else on the host by the
    oracle's restatement of the same generator (bit-identical,
    tests/test_gpu_atsize.py), so the CPU reference arm never loads
    libmhsk.so.  Variants: "-twins" (plant_twins), "-planted"
    (plant_deletions: deletions of both phases over several rounds)."""
    from paper_2109_06042_b200 import config_instance, plant_twins
    from paper_2109_06042_b200.generate import COUNTER_CONFIGS, plant_deletions

    t = time.time()
    base, _, variant = config.partition("-")
    if base in COUNTER_CONFIGS:
        if ctx is not None:
            csr, _ = ctx.generate_random(*COUNTER_CONFIGS[base], seed, host=True)
        else:
            import oracle

            csr = oracle.generate_random(*COUNTER_CONFIGS[base], seed)
        if variant == "twins":
            csr = plant_twins(csr, 0.01, 0.01, seed + 1)
        elif variant == "planted":
            csr, _ = plant_deletions(csr, seed + 1)
        elif variant:
            raise ValueError(f"unknown config variant {variant!r}")
    else:
        csr = config_instance(config, seed)
    return csr, time.time() - t


class CpuBaseline:
    """The reference's algorithm on the host cores (oracle port:
    parallel.py:80-161 as bitset AND + popcount with the reference's early
    exits, AVX-512 VPOPCNTDQ when the host has it, all threads).  Each phase
    operand (incidence_matrix + bitsets) is built once and timed; a sample is
    the round-1 decisions of the first J items of each phase at full width K,
    J sized so a phase sample takes ~budget_s / 2 (and occupies every
    thread).  One full round = both builds + the per-item rates x M."""

    def __init__(self, csr, budget_s: float, threads: int = 0):
        import oracle

        self.csr = csr
        self.threads = threads or oracle.threads_available()
        self.simd = "avx512-vpopcntdq" if oracle.simd(-1) else "scalar popcnt"
        self.phases = {w: oracle.PhaseSample(csr, w, self.threads) for w in ("edges", "vertices")}
        self.sizes = {}
        for which, ph in self.phases.items():
            j = min(ph.items, 32 * self.threads)
            while True:
                t0 = time.perf_counter()
                ph.decide(0, j)
                dt = time.perf_counter() - t0
                if dt > budget_s / 8 or j >= ph.items:
                    break
                j = min(ph.items, max(j * 2, int(j * (budget_s / 8) / max(dt, 1e-3))))
            self.sizes[which] = min(ph.items, max(j, int(j * (budget_s / 2) / max(dt, 1e-3))))

    def sample(self) -> dict:
        per_item, total = {}, 0.0
        for which, ph in self.phases.items():
            j = self.sizes[which]
            t0 = time.perf_counter()
            ph.decide(0, j)
            dt = time.perf_counter() - t0
            total += dt
            per_item[which] = dt / j
        build = sum(ph.build_s for ph in self.phases.values())
        est = build + per_item["edges"] * self.csr.m + per_item["vertices"] * self.csr.n
        je, jv = self.sizes["edges"], self.sizes["vertices"]
        text = (f"round-1 decisions of the first {je} edges and {jv} vertices at full width "
                f"(oracle port of parallel.py:80-161, {self.simd}, {self.threads} threads) in "
                f"{total:.1f} s, plus the two phase operands built in {build:.1f} s; one full "
                f"round = builds + per-item rates x {self.csr.m} edges / {self.csr.n} vertices "
                f"(a lower bound for a multi-round kernelization)")
        return {"est_round_s": est, "sample_s": total, "build_s": build, "sample": text,
                "threads": self.threads}


def mapped_repo_libs() -> list[str]:
    """Shared objects of this repo mapped into the process."""
    try:
        maps = open("/proc/self/maps").read().split("\n")
    except OSError:
        return []
    libs = {line.split()[-1] for line in maps if line.endswith(".so") and REPO in line}
    return sorted(os.path.relpath(p, REPO) for p in libs)


def run_reference(args, rank: int) -> None:
    """--impl reference: the reference's algorithm on the host cores (oracle
    port; the reference itself is pure Python and ~1e6x slower).
    Each step is a bounded sample of the workload (CpuBaseline.sample, ~cpu_budget
    seconds); value is the incidence-entries/s rate that sample measures.
    Nothing here loads libmhsk.so."""
    if rank != 0:
        return
    import oracle

    csr, _ = make_instance(args.config, args.seed)
    entries = float(csr.n) * float(csr.m)
    threads = oracle.threads_available()
    base = CpuBaseline(csr, args.cpu_budget, threads)   # operand builds + sample sizing: warm-up
    for _ in range(max(0, args.warmup - 1)):
        base.phases["edges"].decide(0, 8)
    est, sample_s = [], []
    samples = None
    for _ in range(args.steps):
        s = base.sample()
        est.append(s["est_round_s"])
        sample_s.append(s["sample_s"])
        samples = s
    t = statistics.median(est)
    value = entries / t
    line = {
        "impl": "reference",
        "metric": "full-kernelization incidence-entries/s",
        "value": value, "unit": "incidence-entries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(sample_s) * 1e3,
        "ms_per_step_kind": "measured wall time of one step's bounded sample",
        "extrapolated_ms_per_kernelization": t * 1e3,
        "value_kind": ("n*m / (one full round extrapolated from the per-item decision rate "
                       "measured on the sample)"),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64-bitset",
        "data": "synthetic", "config": config_dict(args, csr),
        "cpu_baseline": {"value": value, "unit": "incidence-entries/s", "cores": threads,
                         "kind": "port", "sample": samples["sample"]},
        "e2e": {"value": value, "unit": "incidence-entries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "repo_libs_mapped": mapped_repo_libs(),
    }
    print(json.dumps(line), flush=True)


def ncu_traffic(config: str, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of one Gram launch from
    the newest committed `ncu --set full` capture of this workload and kernel
    variant ("fp4probe": kind::mxf4 with probe pruning, "tc2": kind::i8),
    profiles/r<round>_v<version>_gram_<kernel>_<config>_ncu.txt (also the
    round-1 "r01_final_..." name), if there is one."""
    import glob
    import re

    best = None
    for path in glob.glob(os.path.join(REPO, "profiles", f"r*_gram_{kernel}_{config}_ncu.txt")):
        m = re.match(r"r(\d+)_(?:v(\d+)|final)_gram_", os.path.basename(path))
        if not m:
            continue
        key = (int(m.group(1)), int(m.group(2)) if m.group(2) else 0)
        if best is None or key > best[0]:
            best = (key, path)
    if best is None:
        return None, None
    text = open(best[1]).read()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    total = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        for line in text.splitlines():
            parts = line.split()
            if parts and parts[0] == key:
                total += float(parts[1]) * scale.get(parts[2], 1)
                break
    return (total or None), os.path.relpath(best[1], REPO)


def config_dict(args, csr) -> dict:
    return {"workload": f"{args.config}: {CONFIG_DESC.get(args.config.split('-')[0], args.config)}"
                        + (" + planted twins" if args.config.endswith("-twins") else ""),
            "n": int(csr.n), "m": int(csr.m), "nnz": int(csr.nnz),
            "alpha": int(csr.demand.max()) if csr.m else 0, "seed": args.seed, "rule": "dp",
            "parallelism": f"tile-slices x{args.gpus} + NCCL allreduce of deleter counts",
            "l2": "operand (n*m int8) and CSR larger than L2; 512 MiB L2 flush between steps"}


def secondary_run(ctx, name: str, args, flush) -> dict:
    """Device time of one more config (N=1): same step, same timing rules as
    the headline, reported with its rounds, deletions and pruning so that a
    multi-round, non-vacuous run (the planted variants) is measured too.
    NAME+int8: the same with int8 operands (tcgen05 kind::i8, option fp4=0),
    the metric's "int8 TC util"."""
    import torch

    base, _, variant = name.partition("+")
    csr, gen_s = make_instance(base, args.seed, ctx)
    if variant == "int8":
        ctx.set_option("fp4", 0)
    dev = torch.device("cuda", ctx.device)
    d_ptr = torch.from_numpy(csr.edge_ptr).to(dev)
    d_vtx = torch.from_numpy(csr.edge_vtx).to(dev)
    d_dem = torch.from_numpy(csr.demand).to(dev)
    d_va = torch.empty(max(csr.n, 1), dtype=torch.uint8, device=dev)
    d_ea = torch.empty(max(csr.m, 1), dtype=torch.uint8, device=dev)

    def step():
        return ctx.kernelize_device(csr.n, csr.m, d_ptr.data_ptr(), d_vtx.data_ptr(),
                                    d_dem.data_ptr(), d_va.data_ptr(), d_ea.data_ptr())

    for _ in range(max(1, min(args.warmup, 2))):
        step()
    stats = []
    for _ in range(max(1, min(args.steps, 3))):
        flush.fill_(1)
        torch.cuda.synchronize()
        stats.append(step())
    ms = statistics.mean(s["ms_total"] for s in stats)
    s0 = stats[-1]
    gram_s = s0["ms_gram"] / 1e3
    fp4 = s0.get("fp4_gram_launches", 0) >= s0["gram_launches"] / 2
    out = {"config": name, "n": int(csr.n), "m": int(csr.m), "nnz": int(csr.nnz),
           "ms_per_step": ms, "value": float(csr.n) * float(csr.m) / (ms / 1e3),
           "unit": "incidence-entries/s", "steps": len(stats), "rounds": int(s0["rounds"]),
           "deleted": {"dp": int(s0["deleted_edges"]), "md": int(s0["deleted_vertices"])},
           "gram_ms": s0["ms_gram"], "gram_share_of_step": s0["ms_gram"] / ms if ms else 0.0,
           "gram_achieved": (s0["executed_ops"] / gram_s / 1e12) if gram_s > 0 else 0.0,
           "gram_peak": 9000.0 if fp4 else 4500.0,
           "gram_unit": "TFLOP/s (fp4)" if fp4 else "TOPS (int8)",
           "executed_ops": int(s0["executed_ops"]), "algorithmic_ops": int(s0["gram_ops"]),
           "pruned_ops_frac": (1.0 - s0["executed_ops"] / s0["gram_ops"]) if s0["gram_ops"] else 0.0,
           "pruned_tiles": int(s0["pruned_tiles"]), "verified_pairs": int(s0["verified_pairs"]),
           "gpu_launches": int(sum(s["kernel_launches"] for s in stats)), "generate_s": gen_s}
    out["gram_frac"] = out["gram_achieved"] / out["gram_peak"]
    if variant == "int8":
        ctx.set_option("fp4", 1)
    del d_ptr, d_vtx, d_dem, d_va, d_ea
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--backend", default="tc", choices=["tc", "tc1", "simt"])
    ap.add_argument("--cpu-budget", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--secondary", default="auto",
                    help="comma-separated extra configs timed at N=1 and reported under "
                         "'secondary' (auto: c4+int8,c4-planted,c5-planted for the c4 headline; none;"
                         " NAME+int8: int8 operands)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    from paper_2109_06042_b200 import _native

    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    ctx = _native.Context(local_rank, backend=args.backend)
    csr, gen_s = make_instance(args.config, args.seed, ctx)
    entries = float(csr.n) * float(csr.m)

    if world > 1:
        from paper_2109_06042_b200.dist import TorchDistAllreduce

        ctx.set_shard(rank, world, TorchDistAllreduce(local_rank))

    dev = torch.device("cuda", local_rank)
    d_ptr = torch.from_numpy(csr.edge_ptr).to(dev)
    d_vtx = torch.from_numpy(csr.edge_vtx if csr.nnz else np.zeros(1, np.int32)).to(dev)
    d_dem = torch.from_numpy(csr.demand if csr.m else np.zeros(1, np.int32)).to(dev)
    d_va = torch.empty(max(csr.n, 1), dtype=torch.uint8, device=dev)
    d_ea = torch.empty(max(csr.m, 1), dtype=torch.uint8, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    def step():
        return ctx.kernelize_device(csr.n, csr.m, d_ptr.data_ptr(), d_vtx.data_ptr(),
                                    d_dem.data_ptr(), d_va.data_ptr(), d_ea.data_ptr())

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
        flush.fill_(1)
    barrier()
    stats = []
    with ClockSampler(local_rank) as clocks:
        barrier()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            stats.append(step())
        barrier()
        wall = time.perf_counter() - w0
    dev_ms = [s["ms_total"] for s in stats]
    ms_step = statistics.mean(dev_ms)
    if world > 1:
        t = torch.tensor([ms_step], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    value = entries / (ms_step / 1e3)

    # ---- end to end through the host-pointer C ABI (pinned buffers)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    from paper_2109_06042_b200.instance import CSRInstance

    hcsr = CSRInstance(csr.n, pin(csr.edge_ptr), pin(csr.edge_vtx), pin(csr.demand), validate=False)
    e2e_stats = []
    # warm the host path -- and the PCIe link: a fresh process sees the first
    # seconds of host->device copies at ~50 instead of ~55 GB/s (same box,
    # tools/e2e_trace.py), so calls continue for >= 1 s before timing
    t_warm = time.perf_counter()
    for i in range(200):
        ctx.kernelize(hcsr)
        if i >= 2 and time.perf_counter() - t_warm > 1.0:
            break
    barrier()
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        e2e_stats.append(ctx.kernelize(hcsr)[2])
    barrier()
    e2e_ms = statistics.mean(s["ms_total"] for s in e2e_stats)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    # this box's pinned host -> device bandwidth for the same member array (a
    # plain copy, CUDA events): the e2e floor the upload alone sets
    h2d_src = torch.from_numpy(hcsr.edge_vtx)
    h2d_dst = torch.empty(h2d_src.numel(), dtype=torch.int32, device=dev)
    h2d_ms = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h2d_dst.copy_(h2d_src, non_blocking=True)
        e1.record()
        e1.synchronize()
        h2d_ms.append(e0.elapsed_time(e1))
    del h2d_dst
    h2d_gbs = h2d_src.numel() * 4 / (min(h2d_ms) / 1e3) / 1e9

    # ---- roofline of the dominant kernel (tcgen05 Gram product)
    s0 = stats[-1]
    peaks = load_peaks()
    bf16 = peaks.get("bf16_tflops")
    # MEASURED_PEAKS.json has no fp4 / int8 figure: the denominators are the
    # B200 dense datasheet peaks (B200_PROFILING.md: fp4 9 PFLOP/s, int8 4.5
    # POPS), which the on-box microbenchmarks reproduce (tools/mxf4_probe.cu:
    # 8911-8927 TFLOP/s, profiles/r01_mma_peak_fp4.json; tools/mma_peak.cu:
    # 4558-4608 TOPS, profiles/r01_mma_peak_int8.json).
    fp4_run = s0.get("fp4_gram_launches", 0) > 0 and s0["fp4_gram_launches"] >= s0["gram_launches"] / 2
    peak = 9000.0 if fp4_run else 4500.0
    gram_s = s0["ms_gram"] / 1e3
    # tensor work: the algorithmic SYRK count, unless exact pruning skipped
    # MMAs -- probe pruning (dense tiles stopped after a short K prefix that
    # proves no pair can fire) or block-sparse k-block masks.  Then the ops
    # actually issued are the achieved figure and the algorithmic rate is
    # reported separately as "effective" (pruning is disclosed,
    # not counted as algorithmic).
    pruned = 0 < s0["executed_ops"] < 0.9 * s0["gram_ops"]
    pruning = (None if not pruned else "probe" if s0.get("pruned_tiles", 0) > 0 else "block-sparse")
    tensor_ops = s0["executed_ops"] if pruned else s0["gram_ops"]
    achieved = (tensor_ops / gram_s / 1e12) if gram_s > 0 else 0.0
    gram_share = s0["ms_gram"] / s0["ms_total"] if s0["ms_total"] else 0.0
    traffic, traffic_src = ncu_traffic(args.config, "fp4probe" if fp4_run and s0.get("pruned_tiles", 0) > 0
                                       else "tc2" if not fp4_run else "fp4")

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    secondary = []
    names = (["c4+int8", "c4-planted", "c5-planted"] if args.secondary == "auto" and args.config == "c4"
             else [] if args.secondary in ("auto", "none", "") else args.secondary.split(","))
    if world == 1:
        del d_ptr, d_vtx, d_dem, hcsr
        for name in names:
            secondary.append(secondary_run(ctx, name, args, flush))

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        s = CpuBaseline(csr, args.cpu_budget).sample()
        cpu = {"value": entries / s["est_round_s"], "unit": "incidence-entries/s",
               "cores": s["threads"], "kind": "port", "sample": s["sample"]}

    line = {
        "metric": "full-kernelization incidence-entries/s",
        "value": value,
        "unit": "incidence-entries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": ("fp4 e2m1 (0/1 incidence, exact f32 accumulation, counts < 2^24)" if fp4_run
                  else "int8 (0/1 incidence, exact int32 accumulation)"),
        "data": "synthetic",
        "config": config_dict(args, csr),
        "rounds": int(s0["rounds"]),
        "deleted": {"dp": int(s0["deleted_edges"]), "md": int(s0["deleted_vertices"])},
        "gpu_launches": int(sum(s["kernel_launches"] for s in stats)),
        "e2e": {"value": entries / (e2e_ms / 1e3), "unit": "incidence-entries/s",
                "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(e2e_stats[-1]["h2d_bytes"]),
                "d2h_bytes_per_step": int(e2e_stats[-1]["d2h_bytes"]),
                "pcie_h2d_gbs": h2d_gbs, "member_copy_ms": min(h2d_ms),
                "ms_steps": [round(s["ms_total"], 3) for s in e2e_stats]},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s (fp4)" if fp4_run else "TOPS (int8)", "frac": achieved / peak,
                     "traffic": traffic, "traffic_unit": "bytes per launch (DRAM read+write)",
                     "traffic_source": traffic_src,
                     "kernel": ("gram_tc2_kernel<FP4> (tcgen05.mma.cta_group::2.kind::mxf4.block_scale, "
                                "fused predicates)" if fp4_run else
                                "gram_tc2_kernel (tcgen05.mma.cta_group::2.kind::i8, fused predicates)"),
                     "peak_source": ("B200 dense fp4 9 PFLOP/s (B200_PROFILING.md); on-box tcgen05 kind::mxf4 "
                                     "microbenchmark 8911-8927 TFLOP/s (profiles/r01_mma_peak_fp4.json); "
                                     "MEASURED_PEAKS.json has bf16 only" if fp4_run else
                                     "B200 dense int8 datasheet 4500 TOPS; on-box tcgen05 kind::i8 "
                                     "microbenchmark 4558-4608 TOPS (profiles/r01_mma_peak_int8.json); "
                                     "MEASURED_PEAKS.json has bf16 only"),
                     "frac_of_measured_bf16_x": ((achieved / ((4.0 if fp4_run else 2.0) * bf16)) if bf16 else None),
                     "gram_share_of_step": gram_share,
                     "executed_ops": int(s0["executed_ops"]), "algorithmic_ops": int(s0["gram_ops"]),
                     "pruning": pruning, "pruned_tiles": int(s0.get("pruned_tiles", 0)),
                     "pruned_ops_frac": (1.0 - s0["executed_ops"] / s0["gram_ops"]) if s0["gram_ops"] else 0.0},
        "cpu_baseline": cpu,
        "secondary": secondary,
        "clocks": clocks.summary(),
        "wall_s_timed_region": wall,
        "generate_s": gen_s,
        "backend": args.backend,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
