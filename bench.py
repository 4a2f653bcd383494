"""BinSketch hot-path benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload large|medium|ranking|buildonly|tiny] [--no-extras] [--no-cpu-baseline]

Default workload = BASELINE.json configs[4] ("Large"): one step is the whole
hot path on synthetic Zipf CSR already resident in HBM:
  a1 make_pi (d = 500,000) -> a2 build 200,000 sketches (N = 1024) ->
  a3 popcounts -> a4/a5/a6 all-pairs AND-popcount + fp64 IP estimate ->
  a7 top-50 per row (self-join, self excluded).
value = estimated pairs/s (4e10 ordered pairs per step per GPU). The
build-only HBM measurement (configs[3]) is reported in "build".

Multi-GPU (torchrun): every rank runs an independent problem instance (its
own data seed) with no data-path collective; value = all ranks' pairs / max
rank time ("scaling": "weak").

--impl reference: the CPU oracle (oracle/, the reference arm of this tier)
timed on the host cores on a bounded sample of the same workload.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "sketch rows/s (HBM GB/s) and estimated pairs/s vs popc roofline, 1xB200"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
SM_COUNT_B200 = 148
# K9 (tools/microbench.cu, profiles/r02_microbench_k9.jsonl): POPC per SM clock, median over SMs of
# ops / busy span by clock64 (clock-independent), median of 3 runs, SM clock verified near max
# (implied 1942 MHz). The CUDA guide's table value is 16.
POPC_PER_CLK_SM = 15.11
POPC_BASIS = "K9 measured 15.11 POPC/clk/SM (profiles/r02_microbench_k9.jsonl) x 148 SMs x SM clock"
# ncu --set full of the fused top-k kernel at this workload (one launch).
INT8_NOMINAL_TOPS = 4500.0   # B200 dense int8 tensor peak (datasheet; the guide's 4.5 POPS) — context beside the measured basis
TOPK_NCU = {"source": "profiles/r02_final6/topk_large_summary.txt", "tensor_pipe_active_pct": 45.9,
            "issue_active_pct": 21.4, "dram_bytes_per_launch": 1.464e9 + 0.576e9, "kernel_share_of_stage": "98.4 %",
            "launch_list": "profiles/r02_final6/launches_large_summary.txt"}
# Ranking: the dominant kernel of the top-k call is the tensor-core AND-popcount with the integer
# screen in its epilogue (tc_pairs_kernel<kTcScreen>, K4d). Its share of the call's
# critical path from the committed launch list (cold-cache, serialised, ms per call): popcounts
# 0.0168; then max(sample branch: query + sample widening ~0.010, sample AND-popcount 0.0205, range
# 0.0045, thresholds 0.0666 = 0.1016; db branch on the second stream: popcount sort 0.0475, db
# widening ~0.110 = 0.158); screen 0.2237; list top-k 0.1071 -> 0.506 ms, screen share 0.442.
RANK_NCU = {"source": "profiles/r02_tc_screen_summary.txt", "kernel_share_of_stage": 0.2237 / 0.506,
            "dram_bytes_per_launch": 431.3e6 + 25.7e6, "tensor_pipe_active_pct": 93.2,
            "launch_list": "profiles/r02_launches_ranking_summary.txt"}
HBM_FALLBACK_GBS = 6650.0     # B200_PROFILING.md fallback


# ----------------------------------------------------------------- utils --
def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": HBM_FALLBACK_GBS, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        # NVML polling every 5 ms (starts in microseconds, so short timed regions are covered);
        # the nvidia-smi loop is the fallback
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.thread = threading.Thread(target=self._poll_nvml, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 1.0:
                time.sleep(0.001)
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _poll_nvml(self):
        nv = self.nvml
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
                smax = nv.nvmlDeviceGetMaxClockInfo(self.handle, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                flags = ["Active" if (r & b) else "Not Active" for b in bits.values()]
                self.lines.append(", ".join([str(self.gpu), str(sm), str(smax), "0", hex(r)] + flags))
            except Exception:
                pass
            time.sleep(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.thread.join(timeout=1.0)
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = max(smax, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------- workloads --
def workload_spec(name):
    import synth
    if name == "large":
        return dict(db=synth.LARGE, q=None, N=synth.LARGE_N, k=synth.LARGE_K, measure=1, exclude_self=True,
                    desc="configs[4] Large: n=200000 sketches N=1024 from d=500000 CSR (lognormal mean 100, "
                         "Zipf 1.1); build + self-join IP top-50 (self excluded)")
    if name == "ranking":
        return dict(db=synth.RANKING_DB, q=synth.RANKING_Q, N=synth.RANKING_N, k=synth.RANKING_K, measure=4,
                    measures=(4, 8), exclude_self=False,
                    desc="configs[2] Ranking: db 100000 + 1000 queries, d=102660, N=4096; build + JS top-100 "
                         "+ COS top-100 (pairs counted once per measure)")
    if name == "tiny":
        return dict(db=synth.TINY, q=None, N=synth.TINY_N, k=10, measure=4, exclude_self=True,
                    desc="configs[0] Tiny: n=1000, d=5000, N=1224; build + JS top-10")
    raise ValueError(name)


def max_over_ranks(x: float, ws: int, device: str = "cuda") -> float:
    """MAX of a per-rank scalar over the process group (plumbing only: NCCL on GPUs, gloo on CPU)."""
    if ws <= 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def csr_sha256(ip_h, ix_h, qp_h=None, qx_h=None) -> str:
    """sha256(indptr || indices [|| query indptr || query indices]) of the workload's synthetic CSR
    (the inputs are identified by hash in every bench line)."""
    import hashlib
    h = hashlib.sha256(ip_h.tobytes())
    h.update(ix_h.tobytes())
    if qp_h is not None:
        h.update(qp_h.tobytes())
        h.update(qx_h.tobytes())
    return h.hexdigest()


def aggregate_value(ws: int, units_per_rank_step: int, steps: int, t_max: float) -> float:
    """Whole-job throughput: all ranks' units over the slowest rank's time (weak scaling)."""
    return ws * units_per_rank_step * steps / t_max


def rank_spec(spec, rank):
    import synth
    if rank == 0:
        return spec
    return synth.CSRSpec(**{**spec.__dict__, "seed": spec.seed + 1000 * rank})


# ------------------------------------------------------------- our arm ----
def run_ours(args):
    import torch
    import torch.distributed as dist

    import synth
    from paper_1910_04658_b200 import binsketch as bs

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pk, pk_src = peaks()

    w = workload_spec(args.workload)
    db_spec = rank_spec(w["db"], rank)
    N, k, measure = w["N"], w["k"], w["measure"]
    d = db_spec.d
    W = (N + 31) // 32
    ip_h, ix_h = synth.make_csr(db_spec)
    n = db_spec.n
    ip = torch.from_numpy(ip_h).cuda()
    ix = torch.from_numpy(ix_h).cuda()
    if w["q"] is not None:
        qp_h, qx_h = synth.make_csr(rank_spec(w["q"], rank))
        qp, qx = torch.from_numpy(qp_h).cuda(), torch.from_numpy(qx_h).cuda()
        nq = w["q"].n
    else:
        qp_h = qx_h = qp = qx = None
        nq = n
    pi = torch.empty(d, dtype=torch.int32, device="cuda")
    sk = torch.empty((n, W), dtype=torch.int32, device="cuda")
    qsk = torch.empty((nq, W), dtype=torch.int32, device="cuda") if qp is not None else None
    mmask = 0
    for m_ in w.get("measures", (measure,)):
        mmask |= m_
    nplanes = bin(mmask).count("1")
    oshape = (nq, k) if nplanes == 1 else (nplanes, nq, k)
    out_idx = torch.empty(oshape, dtype=torch.int32, device="cuda")
    out_score = torch.empty(oshape, dtype=torch.float32, device="cuda")
    wsp = torch.empty(max(1, bs.workspace_bytes(bs.OP_TOPK, nq, n, N, k)), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")   # > 126 MB L2
    stream = torch.cuda.current_stream()
    nnz = int(ip_h[-1])

    ev = {name: [] for name in ("step", "build", "topk")}

    def step(record):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if record else None
        if record:
            e[0].record(stream)
        bs.make_pi(synth.PI_SEED, d, N, out=pi)
        bs.build(pi, d, N, ip, ix, out=sk)
        if qp is not None:
            bs.build(pi, d, N, qp, qx, out=qsk)
        if record:
            e[1].record(stream)
        # all the workload's measures in one call (one AND-popcount table for all of them)
        bs.topk(qsk if qsk is not None else sk, sk, N, d, mmask, k, exclude_self=w["exclude_self"],
                out_idx=out_idx, out_score=out_score, ws=wsp)
        if record:
            e[2].record(stream)
            ev["step"].append((e[0], e[2]))
            ev["build"].append((e[0], e[1]))
            ev["topk"].append((e[1], e[2]))

    for _ in range(args.warmup):
        step(False)
    bs.device_status()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = bs.launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()                          # L2 flush between timed steps (outside the events)
            step(True)
        torch.cuda.synchronize()
    launches = bs.launch_count() - l0 - 0
    bs.device_status()

    def tot(name):
        return sum(a.elapsed_time(b) for a, b in ev[name]) * 1e-3     # seconds over K steps

    t_step, t_build, t_topk = tot("step"), tot("build"), tot("topk")
    t_max = max_over_ranks(t_step, ws)
    pairs_per_step = nq * n * len(w.get("measures", (measure,)))   # ordered pairs scored per measure pass
    value = aggregate_value(ws, pairs_per_step, args.steps, t_max)
    clocks = clk.summary()

    # --- e2e: host (pinned) CSR -> build -> top-k -> host results, through the public API ---
    e2e = None
    ip_pin = torch.from_numpy(ip_h).pin_memory()
    ix_pin = torch.from_numpy(ix_h).pin_memory()
    qp_pin = torch.from_numpy(qp_h).pin_memory() if qp_h is not None else None
    qx_pin = torch.from_numpy(qx_h).pin_memory() if qx_h is not None else None
    pi_pin = torch.empty(d, dtype=torch.int32).pin_memory()
    pi_pin.copy_(pi.cpu())
    bufs = {}
    ms_e2e = w.get("measures", (measure,))
    batch = (ip_pin, ix_pin) if qp_pin is None else (ip_pin, ix_pin, qp_pin, qx_pin)

    def e2e_run(nsteps):
        # nsteps batches through the streaming host-CSR call: every batch copies its own CSR (and pi)
        # in and its own lists out; batch i+1's upload and batch i's download overlap the compute
        return bs.topk_from_host_csr_batches([batch] * nsteps, pi_pin, d, N, ms_e2e, k,
                                             exclude_self=w["exclude_self"], bufs=bufs,
                                             before_batch=lambda i: flush.zero_())

    e2e_run(max(1, args.warmup))
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    h2d, d2h = e2e_run(args.steps)
    b.record(stream)
    b.synchronize()
    tsum = max_over_ranks(a.elapsed_time(b) * 1e-3, ws)
    e2e = {"value": aggregate_value(ws, pairs_per_step, args.steps, tsum), "unit": "pairs/s",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "pipeline": "steps streamed: step i+1's H2D and step i's D2H overlap the compute (copy stream); "
                       "L2 flushed before every step inside the timed region"}
    del bufs

    # --- roofline of the dominant kernel ---
    # Default engine: tensor cores (tc_pairs_kernel, fused top-k: tcgen05 kind::i8 on {0,1}-byte
    # operands + fp64 top-k epilogue). Algorithmic work = 2 * pairs * N int8 ops (the K padding to
    # a multiple of 128 is overhead, not credit). Peak = int8 dense = 2 x the measured bf16 cuBLAS
    # peak (nominal int8 : bf16 = 4.5 : 2.25): the BURST figure, because these steps run ~40 ms at
    # the maximum SM clock with no power cap (clocks below); the sustained figure (measured
    # power-capped at 1342 MHz) is printed beside it. Time basis = the whole top-k call (popcounts,
    # sort, expansion, the kernel, merge), so frac is a lower bound for the kernel itself.
    path = bs.topk_path(nq, n, N, d, k)    # the kernel path of this call (binsketch_topk_path)
    f_sm = (clocks["sm_mhz"] or pk.get("sm_max_mhz", 1965.0)) * 1e6
    peak_words = SM_COUNT_B200 * POPC_PER_CLK_SM * f_sm              # word-ops/s at the measured clock
    achieved_words = pairs_per_step * W * args.steps / t_topk
    popc = {"achieved": achieved_words / 1e12, "peak": peak_words / 1e12, "unit": "Tword-popc/s",
            "frac": achieved_words / peak_words, "peak_basis": POPC_BASIS + " (measured during this run)"}
    burst = 2.0 * pk.get("bf16_tflops", 1590.0)
    sust = 2.0 * pk.get("bf16_tflops_sustained", pk.get("bf16_tflops", 1590.0))
    ach = 2.0 * pairs_per_step * N * args.steps / t_topk / 1e12
    tc_common = {"achieved": ach, "peak": burst, "unit": "TOPS (int8)", "frac": ach / burst,
                 "peak_basis": "2 x MEASURED_PEAKS bf16_tflops (burst; nominal int8:bf16 = 2:1)",
                 "peak_sustained": sust, "frac_of_sustained": ach / sust,
                 "peak_sustained_basis": "2 x MEASURED_PEAKS bf16_tflops_sustained (power-capped, 1342 MHz)",
                 "peak_nominal": INT8_NOMINAL_TOPS, "frac_of_nominal": ach / INT8_NOMINAL_TOPS,
                 "peak_nominal_basis": "B200 datasheet dense int8 (context: our screen kernel exceeds the bf16-derived basis)",
                 "traffic": None, "popc_equivalent": popc}
    if path == "tc_fused":
        roofline = {"bound": "tensor", "kernel": "tc_pairs_kernel (tcgen05.mma kind::i8, query tile in TMEM + fused top-k)",
                    **tc_common,
                    "time_basis": "whole top-k call (popcount + sort + expand + fused kernel + merge); the kernel's "
                                  "share of it: " + str(TOPK_NCU["kernel_share_of_stage"]) + " (" + TOPK_NCU["launch_list"] + ")"}
        if args.workload == "large":
            roofline["ncu"] = {k_: v for k_, v in TOPK_NCU.items() if k_ != "dram_bytes_per_launch"}
            roofline["traffic"] = TOPK_NCU["dram_bytes_per_launch"]
            roofline["traffic_unit"] = "DRAM bytes per launch (ncu; operands are L2-resident)"
    elif path in ("tc_screen", "tc_pab"):
        # k > 64 or N > 6143: sample thresholds, the tensor-core AND-popcount with the integer screen
        # in its epilogue (survivor lists), the exact list top-k. The screen kernel dominates; its
        # work is the whole contraction (2 * pairs * N int8 ops per measure set), time = the live
        # top-k stage time x its launch-list share.
        share = RANK_NCU["kernel_share_of_stage"]
        pairs_once = nq * n   # the contraction runs once for every requested measure
        ach_k = 2.0 * pairs_once * N * args.steps / (t_topk * share) / 1e12
        roofline = {"bound": "tensor", "kernel": "tc_pairs_kernel<kTcScreen> (AND-popcount + integer screen epilogue; DESIGN.md K4d)",
                    "achieved": ach_k, "peak": burst, "unit": "TOPS (int8)", "frac": ach_k / burst,
                    "peak_basis": "2 x MEASURED_PEAKS bf16_tflops (burst)", "peak_sustained": sust,
                    "peak_nominal": INT8_NOMINAL_TOPS, "frac_of_nominal": ach_k / INT8_NOMINAL_TOPS,
                    "frac_of_sustained": ach_k / sust, "traffic": RANK_NCU["dram_bytes_per_launch"],
                    "traffic_unit": "DRAM bytes per launch (ncu --set full): the widened db operand once",
                    "ncu_tensor_pipe_active_pct": RANK_NCU["tensor_pipe_active_pct"],
                    "time_basis": "live top-k stage time x the kernel's share of the call's critical path in the launch list ("
                                  + RANK_NCU["launch_list"] + "): " + f"{share:.3f}",
                    "whole_call": {"achieved": 2.0 * pairs_once * N * args.steps / t_topk / 1e12, "unit": "TOPS (int8)",
                                   "frac_of_burst": 2.0 * pairs_once * N * args.steps / t_topk / 1e12 / burst,
                                   "time_basis": "whole top-k call (popcounts, sort, expand, sample thresholds, screen, list top-k)"}}
    else:
        # the CUDA-core kernels (BINSKETCH_ENGINE=cuda, or a small call: binsketch_topk_path)
        roofline = {"bound": "alu", "kernel": "topk_kernel (LOP3+POPC mainloop + fp64 epilogue)",
                    "achieved": popc["achieved"], "peak": popc["peak"], "unit": "Tword-popc/s", "frac": popc["frac"],
                    "peak_basis": popc["peak_basis"], "traffic": None}

    result = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32 sketches -> u8 {0,1} tensor-core operands, s32 accumulate, fp64 estimator",
        "data": "synthetic (seeded Zipf-feature CSR, synth/; stands in for the paper's UCI corpora)",
        "config": {"workload": args.workload, "desc": w["desc"], "n": n, "nq": nq, "d": d, "N": N, "k": k,
                   "nnz": nnz, "measure": measure, "pairs_per_step": pairs_per_step,
                   "l2": "flushed between timed steps (256 MB write outside the events)",
                   "parallelism": f"independent instances x{ws} (no data-path collective)",
                   "input_sha256": csr_sha256(ip_h, ix_h, qp_h, qx_h)},
        "stages_ms_per_step": {"build": t_build / args.steps * 1e3, "topk": t_topk / args.steps * 1e3},
        "build_rows_per_s": (n + (nq if qp is not None else 0)) * args.steps / t_build,
        "roofline": roofline, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
        "peaks_source": pk_src,
    }

    if rank == 0 and not args.no_extras and args.workload == "large":
        result["build"] = bench_buildonly(args, bs, torch, pk, pk_src)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        gpu_idx = out_idx.cpu().numpy()
        result["cpu_baseline"], result["parity"] = cpu_baseline(args, w, ip_h, ix_h, qp_h, qx_h, gpu_idx)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def bench_buildonly(args, bs, torch, pk, pk_src):
    """configs[3]: 1e7 rows, d=2^20, N=1024: sketch rows/s and HBM GB/s vs the measured copy peak."""
    import synth
    spec, N = synth.BUILD_ONLY, synth.BUILD_ONLY_N
    ip_h, ix_h = synth.make_csr(spec)
    ip, ix = torch.from_numpy(ip_h).cuda(), torch.from_numpy(ix_h).cuda()
    del ix_h
    n, d, W = spec.n, spec.d, (N + 31) // 32
    nnz = int(ip_h[-1])
    pi = bs.make_pi(synth.PI_SEED, d, N)
    out = torch.empty((n, W), dtype=torch.int32, device="cuda")
    res = {}
    alg_bytes = 4 * nnz + 8 * (n + 1) + 4 * W * n + 4 * d
    for variant in ("table", "seeded"):
        def call():
            if variant == "table":
                bs.build(pi, d, N, ip, ix, out=out)
            else:
                bs.build_seeded(synth.PI_SEED, d, N, ip, ix, out=out)
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        ts = []
        for _ in range(max(5, args.steps)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        t = statistics.median(ts)
        gbs = alg_bytes / t / 1e9
        res[variant] = {"ms": t * 1e3, "rows_per_s": n / t, "hbm_gbs": gbs,
                        "frac_of_measured_hbm": gbs / pk["hbm_gbs"], "frac_of_8TBs_datasheet": gbs / 8000.0}
    bs.device_status()
    res["config"] = {"workload": "buildonly (configs[3])", "n": n, "d": d, "N": N, "nnz": nnz,
                     "algorithmic_bytes": alg_bytes, "bytes_formula": "4*nnz + 8*(n+1) + 4*W*n + 4*d",
                     "peak_gbs": pk["hbm_gbs"], "peak_source": pk_src,
                     "l2": "inputs 3.9 GB >> L2 (no flush needed)"}
    del ip, ix, out
    torch.cuda.empty_cache()
    return res


def _oracle_sample_step(w, ip_h, ix_h, qp_h, qx_h, nsample, nthreads):
    """One bounded oracle step: pi + sketches of all rows + top-k for `nsample` queries vs all rows."""
    import oracle
    import synth
    N, d, k = w["N"], w["db"].d, w["k"]
    pi = oracle.make_pi(synth.PI_SEED, d, N)
    D, _ = oracle.sketch(pi, d, N, ip_h, ix_h)
    if qp_h is not None:
        Q, _ = oracle.sketch(pi, d, N, qp_h, qx_h)
        Q = Q[:nsample]
        oracle.topk(Q, D, N, d, w["measure"], k, exclude_self=False, nthreads=nthreads)
    else:
        oracle.topk(D[:nsample], D, N, d, w["measure"], k, exclude_self=w["exclude_self"], nthreads=nthreads)
    return nsample * D.shape[0]


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _omp_threads(n):
    """Thread count of the oracle's OpenMP runtime (libgomp is shared with liboracle.so)."""
    import ctypes
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
        return True
    except OSError:
        return False


def cpu_baseline(args, w, ip_h, ix_h, qp_h, qx_h, gpu_idx):
    """The CPU oracle (as it stands, never tuned) on the GPU box's host cores, bounded samples of
    the same workload: top-k pairs/s all cores and one thread, sketch rows/s all cores and one
    thread, median of 3 each. The all-core top-k lists double as the in-run parity check of the
    GPU's lists for the same query rows (this leg is the one place the bench may run the oracle)."""
    import oracle
    import synth
    N, d, k, m = w["N"], w["db"].d, w["k"], w["measure"]
    cores = os.cpu_count() or 1
    nq_all = {"large": 1000, "ranking": 100, "tiny": 1000}[args.workload]
    nq_one = {"large": 50, "ranking": 5, "tiny": 100}[args.workload]
    pi = oracle.make_pi(synth.PI_SEED, d, N)

    def timed(fn, reps=3):
        ts, out = [], None
        for _ in range(reps):
            t0 = time.perf_counter()
            out = fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts), out

    _omp_threads(cores)
    t_sk, (D, _) = timed(lambda: oracle.sketch(pi, d, N, ip_h, ix_h))   # orc_sketch is sequential
    if qp_h is not None:
        Q, _ = oracle.sketch(pi, d, N, qp_h, qx_h)
        excl = False
    else:
        Q, excl = D, w["exclude_self"]
    ndb = D.shape[0]
    t_all, (ri, _) = timed(lambda: oracle.topk(Q[:nq_all], D, N, d, m, k, exclude_self=excl, nthreads=cores))
    t_one, _ = timed(lambda: oracle.topk(Q[:nq_one], D, N, d, m, k, exclude_self=excl, nthreads=1))
    rows = len(ip_h) - 1
    g = gpu_idx if gpu_idx.ndim == 2 else gpu_idx[0]          # first measure's plane
    same = int(np.sum(np.all(g[:nq_all] == ri, axis=1)))
    parity = {"kind": f"top-{k} index lists of query rows 0..{nq_all - 1} (of {g.shape[0]}) from the last timed "
                      "step vs the CPU oracle, bit-exact, ties to the lower index",
              "rows": nq_all, "identical_rows": same, "ok": same == nq_all,
              "full_check": "profiles/r02_parity_large_full.log" if args.workload == "large" else None}
    base = {"value": nq_all * ndb / t_all, "unit": "pairs/s", "cores": cores, "kind": "oracle",
            "cpu_model": _cpu_model(), "repeats": 3, "statistic": "median",
            "single_thread": {"value": nq_one * ndb / t_one, "unit": "pairs/s", "cores": 1},
            "build_rows_per_s": {"value": rows / t_sk, "cores": 1,
                                 "sample": f"oracle sketch of all {rows} rows of this workload's CSR (N={N}); "
                                           "the oracle's sketch loop is sequential (oracle.cpp orc_sketch)"},
            "sample": f"oracle (oracle/oracle.cpp, OpenMP): top-{k} of {nq_all} query rows vs all {ndb} db rows "
                      f"({cores} threads) and of {nq_one} rows (1 thread); median of 3 each"}
    return base, parity


# -------------------------------------------------------- reference arm ---
def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    import synth
    w = workload_spec(args.workload)
    ip_h, ix_h = synth.make_csr(w["db"])
    if w["q"] is not None:
        qp_h, qx_h = synth.make_csr(w["q"])
    else:
        qp_h = qx_h = None
    nthreads = os.cpu_count() or 1
    nsample = {"large": 1000, "ranking": 100, "tiny": 1000}[args.workload]
    for _ in range(args.warmup):
        _oracle_sample_step(w, ip_h, ix_h, qp_h, qx_h, max(1, nsample // 10), nthreads)
    t0 = time.perf_counter()
    pairs = 0
    for _ in range(args.steps):
        pairs += _oracle_sample_step(w, ip_h, ix_h, qp_h, qx_h, nsample, nthreads)
    t = time.perf_counter() - t0
    v = pairs / t
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "pairs/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32/fp64 (CPU)", "data": "synthetic (same seeded generator)",
        "config": {"workload": args.workload, "desc": w["desc"]},
        "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": nthreads, "kind": "oracle",
                         "sample": f"each step: pi + all sketches + top-{w['k']} for {nsample} query rows vs all db rows"},
        "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="large", choices=["large", "ranking", "tiny"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
