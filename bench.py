"""Benchmark: fitness evaluations per second of the p-hub-median hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Workload (BASELINE.json configs[2], URAND-style): instance
generate_urand(1000, 20, 1704, (1, 0.75, 1)), a population of 8192 uniform
20-hub sets per GPU resident in HBM.  One step = score the whole population:
K2 nearest-hub allocation + K3 fitness + finalise (3 kernels).  L2 is flushed
(256 MiB write) between steps, outside the timed events.  With torchrun
(N > 1) every rank scores its own 8192 individuals (weak scaling); the step
time is the max over ranks.

``--gpus N`` without torchrun spawns N ranks itself (one process per GPU,
NCCL), and fails if fewer than N devices are visible; under torchrun the
world size comes from the environment and must equal --gpus.

``--impl reference`` times the reference's algorithm on the host cores (the
numpy restatement in oracle/, bit-pinned to the reference's own outputs) on
the same instance and population: rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fitness evals/sec at n=1000,p=20 (1-8 B200); GA time-to-best-cost vs CPU ref"
KERNEL_NAMES = {
    "tensor-pair": "k_fitness_tcp (K3-TC/P: u8 one-hot GEMM on tcgen05 CTA pairs over the triangular fold of W + integer bins + fused finalise)",
    "tensor-pair-full": "k_fitness_tcp (K3-TC/P on the full W)",
    "fp64": "k_fitness (K3: fp64 smem gather)",
}
N, P, SEED, FACTORS = 1000, 20, 1704, (1.0, 0.75, 1.0)
POP = 8192
HBM_FALLBACK = 6650.0


NCU_TRAFFIC_FILE = "profiles/ncu_traffic_r2.json"


def ncu_traffic(fit_kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum of the K3 launch from one
    committed `ncu --set full` capture of this bench (None when absent)."""
    try:
        with open(Path(__file__).resolve().parent / NCU_TRAFFIC_FILE) as f:
            ks = json.load(f)["kernels"]
    except (OSError, ValueError, KeyError):
        return None
    import re

    pat = {"tensor-pair": r"k_fitness_tcp\b", "tensor-pair-full": r"k_fitness_tcp\b",
           "fp64": r"k_fitness<"}[fit_kernel]
    for name, v in ks.items():
        if re.search(pat, name):
            return v["dram_bytes"]
    return None


def ncu_kernel_record(pattern):
    """The committed ncu record of the first kernel matching `pattern`."""
    import re

    try:
        with open(ROOT / NCU_TRAFFIC_FILE) as f:
            ks = json.load(f)["kernels"]
    except (OSError, ValueError, KeyError):
        return None
    for name, v in ks.items():
        if re.search(pattern, name):
            return v
    return None


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


INT8_PEAK_FILE = "profiles/int8_peak_r2.json"


def peaks_int8():
    """Dense int8 tensor peak measured on this pool's B200 by tools/int8_peak.cu
    (committed result), else 2x the measured bf16 burst (nominal ratio)."""
    try:
        return float(json.loads((ROOT / INT8_PEAK_FILE).read_text())["int8_tops"]), \
            f"measured: tools/int8_peak.cu ({INT8_PEAK_FILE})"
    except Exception:
        try:
            bf16 = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops"])
        except Exception:
            bf16 = 1590.0
        return 2.0 * bf16, "2x measured dense bf16 (int8 microbench result missing)"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# CPU baseline: the oracle restatement of the reference hot functions
# (allocate_to_nearest + _components), one process per core
# ---------------------------------------------------------------------------

_CPU = {}


def _cpu_init():
    from oracle import hm_oracle as orc

    _CPU["pr"] = orc.urand_problem(N, P, SEED, FACTORS)
    _CPU["pop"] = orc.bench_population(N, P, 512)


def _cpu_work(args):
    from oracle import hm_oracle as orc

    start, count = args
    pr, pop = _CPU["pr"], _CPU["pop"]
    t0 = time.perf_counter()
    acc = 0.0
    for k in range(count):
        h = pop[(start + k) % len(pop)]
        a = orc.nearest(pr.C, h)
        c, t, d = orc.cost_terms(pr, h, a)
        acc += c + t + d
    return time.perf_counter() - t0, acc


class CpuBaseline:
    def __init__(self, cores: int | None = None):
        import multiprocessing as mp

        self.cores = cores or os.cpu_count() or 1
        self.pool = mp.get_context("fork").Pool(self.cores, initializer=_cpu_init)
        # calibrate: evals per second per process with every process busy
        self.pool.map(_cpu_work, [(0, 2)] * self.cores)
        t0 = time.perf_counter()
        self.pool.map(_cpu_work, [(0, 8)] * self.cores)
        self.per_core = 8 / (time.perf_counter() - t0)

    def step(self, seconds: float):
        m = max(2, int(self.per_core * seconds))
        t0 = time.perf_counter()
        self.pool.map(_cpu_work, [(r * m, m) for r in range(self.cores)])
        wall = time.perf_counter() - t0
        return self.cores * m, wall, m

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------


class ClockSampler:
    """SM clock and throttle reasons of this rank's GPU, read through NVML.

    ``poll(done)`` samples back to back while the timed kernels run (the host
    has queued every step and waits on the last event), so even a few-ms timed
    region yields samples; a background thread also samples every 2 ms."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, cuda_index: int):
        import threading

        self.h = None
        self.rows = []
        try:
            import pynvml as nv
            import torch

            nv.nvmlInit()
            self.nv = nv
            try:
                pr = torch.cuda.get_device_properties(cuda_index)
                bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
                self.h = nv.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = nv.nvmlDeviceGetHandleByIndex(cuda_index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:
            self.h = None
        self._stop = threading.Event()
        self._t = None
        if self.h is not None:
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()

    def sample(self):
        if self.h is None:
            return
        nv = self.nv
        try:
            mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            return
        self.rows.append((mhz, r))

    def _loop(self):
        while not self._stop.wait(0.002):
            self.sample()

    def poll(self, done) -> None:
        """Sample until done() is true (the timed region's last event)."""
        while not done():
            self.sample()
            time.sleep(0.0002)

    def stop(self):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=1.0)
        if self.h is None or not self.rows:
            return None
        nv = self.nv
        reasons = sorted({name for _, r in self.rows for name, attr in self.REASONS
                          if hasattr(nv, attr) and r & getattr(nv, attr)})
        return {"sm_mhz": statistics.median(m for m, _ in self.rows),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.rows),
                "source": "NVML during the timed region (polled while the queued steps run)"}


# ---------------------------------------------------------------------------
# GA time-to-best-cost vs the CPU reference (BASELINE.json metric, 2nd half)
# ---------------------------------------------------------------------------


def ga_time_to_target(hg, inst, args):
    """The reference's GA (oracle port, one core: the reference `solve` is
    GIL-bound, hm/engine.py:175-177) runs a bounded UR budget; its final best
    cost is the target.  The GPU `solve` with the same GaParams replays the same
    trajectory (same draws, hm/rng.py), so its wall time is the time to reach the
    CPU's best cost.  A larger GPU budget run for at most the CPU's wall time
    shows the best cost the GPU reaches in the same time."""
    from oracle import hm_oracle as orc

    kw = dict(islands=8, pop_size=16, inner_iters=args.ga_inner, outer_iters=1, seed=0)
    params = hg.GaParams(**kw)
    mode = hg.FitnessMode.STANDARD_MILLI
    hg.solve(inst, hg.GaParams(islands=2, pop_size=4, inner_iters=1, outer_iters=1), mode)  # warm
    t0 = time.perf_counter()
    rep = hg.solve(inst, params, mode)
    t_gpu = time.perf_counter() - t0

    pr = orc.Problem(N, P, inst.dist, inst.flow, *FACTORS)
    t0 = time.perf_counter()
    ref = orc.island_ga(pr, kw["islands"], kw["pop_size"], kw["inner_iters"], 1, 0, None, False,
                        "milli")
    t_cpu = time.perf_counter() - t0
    evals = kw["islands"] * kw["pop_size"] * kw["inner_iters"]

    # same wall-clock budget, GPU-sized search: one solve of 128 islands x 64 with
    # as many 25-generation rounds as fit in the CPU reference's time
    t0 = time.perf_counter()
    hg.solve(inst, hg.GaParams(islands=128, pop_size=64, inner_iters=25, outer_iters=1, seed=1),
             mode)
    t_round = time.perf_counter() - t0
    rounds = max(1, int(t_cpu / t_round))
    big = hg.GaParams(islands=128, pop_size=64, inner_iters=25, outer_iters=rounds, seed=1)
    t0 = time.perf_counter()
    rbig = hg.solve(inst, big, mode)
    t_big = time.perf_counter() - t0
    best = rbig.raw_objective
    return {
        "config": f"UR n={N} p={P}, GaParams(islands=8, pop_size=16, inner_iters="
                  f"{kw['inner_iters']}, outer_iters=1, seed=0), milli",
        "cpu_ref_seconds": t_cpu, "cpu_ref_best_raw": ref.raw, "cpu_ref_evals": evals,
        "cpu_ref_kind": "port (oracle/hm_oracle.py island_ga, 1 core)",
        "gpu_seconds_to_target": t_gpu, "gpu_best_raw": rep.raw_objective,
        "gpu_replays_cpu": bool(abs(rep.raw_objective - ref.raw) <= 1e-12 * ref.raw
                                and np.array_equal(rep.best_solution.hubs, ref.hubs)),
        "speedup_time_to_target": t_cpu / t_gpu,
        "gpu_same_wallclock": {"seconds": t_big, "evals": rbig.evaluations, "best_raw": best,
                               "better_than_cpu": bool(best < ref.raw),
                               "trace_milli": list(rbig.trace)[-3:],
                               "config": f"GaParams(islands=128, pop_size=64, inner_iters=25, "
                                         f"outer_iters={rounds}, seed=1)"},
    }


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


SWEEP_NS, SWEEP_PS, SWEEP_BS = (200, 1000, 6000), (5, 20, 50), (4096, 65536)


def sweep(hg, world, rank, barrier):
    """BASELINE configs[4]: fitness-eval throughput over n x p x population per
    GPU (device-resident hub sets, L2 flushed before every evaluation, K2 + K3
    + finalise timed by CUDA events on the instance stream, the max over
    ranks); whole-job evals/s = ranks x B / time, weak scaling."""
    import torch

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = []
    for n in SWEEP_NS:
        for p in SWEEP_PS:
            inst = hg.generate_urand(n, p, SEED, FACTORS, device=True)
            d = inst.device()
            st = torch.cuda.ExternalStream(d.stream)
            for B in SWEEP_BS:
                pop = hg._lib.DevicePopulation(d, B)
                pop.load_hubs(hg.random_population(n, p, B, key=7, start=rank * B)
                              .astype(np.int32))
                reps = 5
                with torch.cuda.stream(st):
                    for _ in range(2):
                        flush.zero_()
                        pop.evaluate(B)
                    barrier()
                    ev = [(torch.cuda.Event(enable_timing=True),
                           torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
                    k3 = []
                    for k in range(reps):
                        flush.zero_()
                        ev[k][0].record(st)
                        pop.evaluate(B)
                        ev[k][1].record(st)
                    barrier()
                    for _ in range(2):
                        flush.zero_()
                        pop.evaluate(B)
                        k3.append(pop.last_fitness_ms())
                ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
                if world > 1:
                    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
                    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                    ms = float(t.item())
                out.append({"n": n, "p": p, "pop_per_gpu": B, "ms": ms,
                            "evals_per_s": world * B / (ms * 1e-3),
                            "k3_ms": float(np.median(k3)), "kernel": d.fitness_kernel})
                del pop
            del inst, d
    return out


def k2_roofline(k2_ms):
    """K2 (nearest-hub allocation) is bound by L1/TEX: its Cq rows (p*n*2 B
    per eval, coalesced) and the fp64 leg gathers (one sector per node);
    frac = ncu's l1tex throughput of the committed capture."""
    rec = ncu_kernel_record(r"k_allocate")
    out = {"kernel": "k_allocate_r (K2: 16-bit pre-filtered argmin, legs, cluster ids)",
           "kernel_ms": k2_ms, "bound": "L1/TEX (gather)",
           "cq_bytes_per_launch": POP * P * N * 2.0}
    if rec:
        out.update({"frac": rec["l1tex_throughput_pct"] / 100.0,
                    "frac_source": f"ncu l1tex__throughput.avg.pct_of_peak_sustained_active, "
                                   f"{NCU_TRAFFIC_FILE}",
                    "traffic": rec["dram_bytes"]})
    return out


def run_gpu(args):
    import torch

    import paper_1704_06258_b200 as hg

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local}, "
                         f"{torch.cuda.device_count()} device(s) visible")
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    hg.set_device(local)

    inst = hg.generate_urand(N, P, SEED, FACTORS)
    dinst = inst.device()
    pop_host = hg.random_population(N, P, POP, key=1, start=rank * POP)
    popd = hg._lib.DevicePopulation(dinst, POP)
    popd.load_hubs(pop_host.astype(np.int32))
    stream = torch.cuda.ExternalStream(dinst.stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            flush.zero_()
            popd.evaluate(POP)
        barrier()
        clocks = ClockSampler(local)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        barrier()
        t_wall0 = time.perf_counter()
        launches0 = hg._lib.launch_count()
        for k in range(args.steps):  # no host sync inside: the GPU stays loaded
            flush.zero_()
            ev[k][0].record(stream)
            popd.evaluate(POP)
            ev[k][1].record(stream)
        launches = hg._lib.launch_count() - launches0
        clocks.poll(ev[-1][1].query)  # clocks while the queued steps run
        barrier()
        t_wall = time.perf_counter() - t_wall0
        clk = clocks.stop()
        step_ms = [a.elapsed_time(b) for a, b in ev]
        # per-launch duration of the dominant kernel (K3), events inside the library
        fit_ms, k2_ms = [], []
        for _ in range(20):
            flush.zero_()
            popd.evaluate(POP)
            fit_ms.append(popd.last_fitness_ms())
            k2_ms.append(popd.last_allocate_ms())

    total_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * POP * args.steps / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps

    # roofline of the dominant kernel (K3 transfer term), per launch
    hbm, hbm_src = peaks()
    fit_kernel = dinst.fitness_kernel
    fit_avg = float(np.mean(fit_ms))
    alg_bytes = POP * (8.0 * N * N + 4.0 * N)
    # K3-TC/P is bound by the int8 tensor pipe: the work is the int8 operations
    # it issues per launch (padding, dummy slots included; on the triangular
    # fold about half of the full contraction's), the peak the measured dense
    # int8 rate of tools/int8_peak.cu
    issued_ops = dinst.mma_ops(POP)
    useful_ops = POP * 2.0 * N * N * P  # the full n x n x p contraction per eval
    int8_peak, int8_src = peaks_int8()
    achieved_tops = issued_ops / (fit_avg * 1e-3) / 1e12
    # every other K3 variant on the same population, for comparison
    variant_ms = {}
    for name in ("fp64", "tensor-pair-full", "tensor-pair"):
        try:
            dinst.set_fitness(hg._lib.FIT_NAMES[name])
        except ValueError:
            continue
        with torch.cuda.stream(stream):
            ms = []
            for _ in range(3):
                flush.zero_()
                popd.evaluate(POP)
                ms.append(popd.last_fitness_ms())
        variant_ms[name] = float(np.median(ms))
    dinst.set_fitness(hg._lib.FIT_AUTO)

    # e2e through the public API with pinned host buffers
    hubs_pin = torch.from_numpy(pop_host).pin_memory().numpy()
    e2e_ms = []
    with torch.cuda.stream(stream):
        for k in range(args.warmup + args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = hg.evaluate_population(inst, hubs_pin)
            dt = time.perf_counter() - t0
            if k >= args.warmup:
                e2e_ms.append(dt * 1e3)
    e2e_total = float(sum(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = world * POP * args.steps / (e2e_total * 1e-3)

    # GA generation throughput (evolve + score) on the UR config, R=128 x pop 64
    ga = hg._lib.DeviceGa(dinst, 128, 0, 128, 64, 3, False, 0)
    seed_hubs = np.sort(inst.middle_rank[:P])
    ga.begin_round(seed_hubs)
    with torch.cuda.stream(stream):
        ga.generations(args.warmup)
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        ga.generations(args.steps)
        g1.record(stream)
        barrier()
        ga_ms = g0.elapsed_time(g1) / args.steps

    # the island GA sharded over every rank: 128 islands x 64 per GPU, champion
    # all_gather (NCCL over NVLink) at each outer-round barrier; wall clock,
    # max over ranks
    gp = hg.GaParams(islands=128 * world, pop_size=64, inner_iters=10, outer_iters=5, seed=1)
    group = torch.distributed.group.WORLD if world > 1 else None
    hg.solve(inst, gp, hg.FitnessMode.STANDARD_MILLI, group=group)  # warm-up: GA objects, NCCL
    barrier()
    t0 = time.perf_counter()
    rep_sh = hg.solve(inst, gp, hg.FitnessMode.STANDARD_MILLI, group=group)
    barrier()
    t_sh = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([t_sh], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_sh = float(tt.item())
    ga_sharded = {"islands": gp.islands, "pop_size": gp.pop_size, "generations": 50,
                  "rounds": gp.outer_iters, "seconds_wall": t_sh,
                  "child_evals_per_s": rep_sh.evaluations / t_sh,
                  "best_raw": rep_sh.raw_objective,
                  "note": "solve(..., group=WORLD) after one warm-up solve of the same shape "
                          "(reused GA objects): islands sharded by global id, one champion "
                          "all_gather per outer round; host loop included"}

    ga_ttt = None
    if rank == 0 and not args.no_cpu:
        ga_ttt = ga_time_to_target(hg, inst, args)

    sweep_pts = sweep(hg, world, rank, barrier) if not args.no_sweep else None

    cpu = None
    if rank == 0 and not args.no_cpu:
        cb = CpuBaseline()
        evals, wall, m = cb.step(args.cpu_seconds)
        cb.close()
        cpu = {"value": evals / wall, "unit": "evals/s", "cores": cb.cores, "kind": "port",
               "sample": f"{cb.cores} processes x {m} evals (allocate_to_nearest + _components "
                         f"restated in numpy, oracle/hm_oracle.py) on the same instance, "
                         f"{wall:.1f} s wall; host CPU {cpu_model()}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "fitness-eval URAND n=1000 p=20, population 8192/GPU "
                                   "(K2 allocation + K3 fitness + finalise)",
                       "n": N, "p": P, "factors": list(FACTORS), "instance_seed": SEED,
                       "pop_per_gpu": POP, "global_pop": POP * world,
                       "parallelism": f"population sharded, {world} rank(s)",
                       "l2": "flushed between steps (256 MiB write, untimed)"},
            "roofline": {"bound": "tensor", "operand": "int8 (tcgen05.mma kind::i8, u8 x u8 -> s32)",
                         "achieved": useful_ops / (fit_avg * 1e-3) / 1e12, "peak": int8_peak,
                         "unit": "TOP/s",
                         "frac": useful_ops / (fit_avg * 1e-3) / 1e12 / int8_peak,
                         "traffic": ncu_traffic(fit_kernel), "traffic_source": NCU_TRAFFIC_FILE,
                         "kernel": KERNEL_NAMES[fit_kernel], "kernel_ms": fit_avg,
                         "algorithmic_ops_per_launch": useful_ops, "peak_source": int8_src,
                         "issued_ops_per_launch": issued_ops,
                         "issued_tops": achieved_tops,
                         "issued_frac": achieved_tops / int8_peak,
                         "note": "achieved = the algorithmic work, 2 n^2 p int8 ops per "
                                 "evaluation (the u8 one-hot contraction of the n x n flows), x "
                                 "the 8192 evaluations of one launch / its event-timed duration; "
                                 "issued = the MMAs the kernel actually runs (the triangular fold "
                                 "of W halves them; padding and dummy slots included)",
                         "k2": k2_roofline(float(np.mean(k2_ms))),
                         "hbm_view": {"alg_bytes_per_launch": alg_bytes,
                                      "alg_gbs": alg_bytes / (fit_avg * 1e-3) / 1e9,
                                      "hbm_peak_gbs": hbm, "peak_source": hbm_src,
                                      "w_reuse_factor": alg_bytes / (fit_avg * 1e-3) / 1e9 / hbm,
                                      "note": "SURVEY 8(d) charges a full fp64 W pass (8n^2+4n B) "
                                              "per eval; W stays on chip across the population, "
                                              "so this ratio is the W-reuse factor, not a "
                                              "roofline fraction"}},
            "kernels_ms": {"k3_selected": fit_kernel, "k3": fit_avg,
                           "k2": float(np.mean(k2_ms)),
                           "k3_variants": variant_ms, "step_total": ms_per_step},
            "e2e": {"value": e2e_value, "unit": "evals/s",
                    "h2d_bytes_per_step": int(pop_host.nbytes),
                    "d2h_bytes_per_step": int(res.nbytes),
                    "api": "paper_1704_06258_b200.evaluate_population (hg_evaluate)"},
            "gpu_launches": launches,
            "clocks": clk,
            "ga": {"child_evals_per_s": world * 128 * 64 / (ga_ms * 1e-3),
                   "ms_per_generation": ga_ms, "config": "R=128 x pop 64 per GPU, strength 3",
                   "launches_per_generation": ga.launches_per_generation,
                   "sharded_solve": ga_sharded},
            "wall_s_timed_region": t_wall,
        }
        if ga_ttt:
            line["ga_time_to_target"] = ga_ttt
        if sweep_pts:
            line["sweep"] = {"what": "BASELINE configs[4]: fitness evals/s over n x p x population "
                                     "per GPU (weak scaling), median of 5 CUDA-event-timed "
                                     "evaluations, L2 flushed before each, max over ranks",
                             "points": sweep_pts}
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------------------
# reference arm: the reference's algorithm on the host cores
# ---------------------------------------------------------------------------


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cb = CpuBaseline()
    # each step is a bounded sample: the whole K + W run stays within ~2.5 min
    per_step = max(0.03, min(args.ref_seconds, 100.0 / (args.steps + args.warmup / 4.0)))
    for _ in range(args.warmup):
        cb.step(per_step / 4)
    evals, walls = 0, 0.0
    m = 0
    for _ in range(args.steps):
        e, w, m = cb.step(per_step)
        evals += e
        walls += w
    cb.close()
    value = evals / walls
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": walls / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": "fitness-eval URAND n=1000 p=20 (allocate_to_nearest + "
                               "_components), bounded sample per step",
                   "n": N, "p": P, "factors": list(FACTORS), "instance_seed": SEED},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cb.cores, "kind": "port",
                         "sample": f"{cb.cores} processes x {m} evals per step; numpy "
                                   f"restatement of hm/model.py:202-207 + "
                                   f"hm/evaluation.py:103-120; host CPU {cpu_model()}"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _spawned_rank(local: int, args, world: int, port: int) -> None:
    os.environ.update(RANK=str(local), LOCAL_RANK=str(local), WORLD_SIZE=str(world),
                      LOCAL_WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    run_gpu(args)


def spawn_ranks(args) -> None:
    """--gpus N outside torchrun: one process per GPU (torch.multiprocessing,
    NCCL), launched here; an error if fewer than N devices are visible."""
    import socket

    import torch
    import torch.multiprocessing as mp

    have = torch.cuda.device_count()
    if have < args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.start_processes(_spawned_rank, args=(args, args.gpus, port), nprocs=args.gpus,
                       start_method="spawn")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--ref-seconds", type=float, default=2.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the configs[4] sweep")
    ap.add_argument("--ga-inner", type=int, default=12,
                    help="generations of the CPU-reference GA run (about 1 s each)")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif "WORLD_SIZE" not in os.environ and args.gpus > 1:
        spawn_ranks(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
