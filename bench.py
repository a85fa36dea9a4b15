#!/usr/bin/env python
"""Benchmark: full FG/BG connected-component labeling + analysis (features, Euler number,
adjacency tree, hole filling) on B200.

Default workload = BASELINE config 2 (the config the metric is quoted on): one step labels the
whole sweep of 105 images of 2048 x 2048, density k/20 (k = 0..20) x granularity
{1, 2, 4, 8, 16}, seed 1.  Inputs are generated on the device with the reference's generator
(bit-identical: tests/test_gpu_generate.py) and stay resident in HBM (440 MB > 126 MB L2, so
no L2 flush is needed between steps).  `--config cfg1|cfg3|cfg4|cfg5` runs the other BASELINE
configs (cfg2 and cfg4 shard their images across ranks, cfg5 splits into strips, cfg1/cfg3 run
one replica per rank).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfgX]

`--gpus N` without torchrun re-launches itself under `torch.distributed.run` with N ranks
(one process per GPU, NCCL).  Batches (cfg2, cfg4) are sharded by image across the ranks --
the image -> rank assignment balances the expected per-image cost (distributed.py) -- so the
total work is fixed (strong scaling); cfg1/cfg3 run one replica per rank; cfg5 is cut into
horizontal strips (strips.py).  Each rank times its own work with CUDA events; time = max
over ranks; value = all ranks' pixels / time.  `--impl reference` times the reference's own
CPU path (oracle/_ref, compiled from the unmodified reference headers) on the host cores,
rank 0 only.

After the timed region every image of the timed batch is compared bit-exactly with the
reference run on the host (`parity` in the JSON line; `--no-parity` skips it).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpixel/s full FG/BG CCA (features+Euler+tree+hole fill); % of HBM roofline"
# concurrent pipelines per large device batch (rl_set_pipelines; the library default 3; env
# RUNLAB_GPU_SPLIT=1 for one pipeline, e.g. for per-kernel profiles of the whole batch)
PIPELINES = int(os.environ.get("RUNLAB_GPU_SPLIT", "3"))
BACKEND = "nccl"  # one process per GPU


# ------------------------------------------------------------------------------ workloads
class Workload:
    """A BASELINE config: image shape, per-image generator specs, sharding."""

    def __init__(self, name: str):
        from paper_2006_09299_b200.runlab import cfg2_cells, cfg4_params
        self.name = name
        if name == "cfg1":
            self.W = self.H = 1024
            self.specs = [("gen", 0.5, 1, 1)]
            self.desc = "cfg1: 1 x 1024x1024, Bernoulli(0.5), g=1, seed 1"
            self.shard = False
        elif name == "cfg2":
            self.W = self.H = 2048
            self.specs = [("gen", d, g, 1) for d, g in cfg2_cells()]
            self.desc = "cfg2: 105 x 2048x2048, density k/20 (k=0..20) x granularity {1,2,4,8,16}, seed 1"
            self.shard = True
        elif name == "cfg3":
            self.W = self.H = 4096
            self.specs = [("rings", 64, 3, 0.02)]
            self.desc = "cfg3: 1 x 4096x4096 nested rings (64x64 blocks, k<=16 rings, 2% salt), seed 3"
            self.shard = False
        elif name == "cfg4":
            self.W, self.H = 1920, 1080
            self.specs = [("gen",) + cfg4_params(i) + (i,) for i in range(4096)]
            self.desc = "cfg4: 4096 x 1920x1080, density U[0.1,0.9], granularity U{1..8}, seed i"
            self.shard = True
        elif name == "cfg5":
            self.W = self.H = 32768
            self.specs = [("gen", 0.45, 4, 5)]
            self.desc = "cfg5: 1 x 32768x32768 (1 Gpixel), Bernoulli(0.45), g=4, seed 5"
            self.shard = False
        else:
            raise SystemExit(f"unknown config {name}")

    def local_specs(self, rank: int, world: int):
        """This rank's images: the whole list for replicated single-image configs, else a
        cost-balanced share of the batch (images are independent)."""
        if not self.shard:
            return self.specs
        from paper_2006_09299_b200.distributed import balanced_shards, image_cost
        costs = [image_cost(s[1], s[2]) for s in self.specs]
        return [self.specs[i] for i in balanced_shards(costs, world)[rank]]

    def make_device(self, specs):
        import torch
        from paper_2006_09299_b200.runlab import generate_device, generate_rings_device
        imgs = torch.empty((len(specs), self.H, self.W), dtype=torch.uint8, device="cuda")
        for i, s in enumerate(specs):
            if s[0] == "gen":
                generate_device(imgs[i].data_ptr(), self.W, self.H, s[1], s[2], s[3])
            else:
                generate_rings_device(imgs[i].data_ptr(), self.W, self.H, s[1], s[2], s[3])
        torch.cuda.synchronize()
        return imgs

    def make_host(self, specs) -> np.ndarray:
        """Same inputs on the host via the oracle's generators (CPU legs only)."""
        from oracle import oracle as O
        out = np.empty((len(specs), self.H, self.W), dtype=np.uint8)
        for i, s in enumerate(specs):
            out[i] = (O.generate(self.W, self.H, s[1], s[2], s[3]) if s[0] == "gen"
                      else O.generate_rings(self.W, self.H, s[1], s[2], s[3]))
        return out

    def cpu_sample(self):
        """Bounded sample for the CPU baseline (timed passes repeat for >= 5 s of wall time)."""
        if self.name == "cfg2":
            return self.specs, "all 105 config-2 images"
        if self.name == "cfg4":
            return self.specs[:64], "the first 64 of the 4096 config-4 images"
        if self.name == "cfg5":
            return None, "1 Gpixel image too large for a bounded sample; see BASELINE.md (3.0 s, 1 core)"
        return self.specs, "the full workload"


def measured_peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def profiled_traffic(config: str, kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu capture of this workload."""
    path = os.path.join(ROOT, "profiles", f"traffic_{config}.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(kernel), os.path.relpath(path, ROOT)
    except Exception:
        return None, None


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu=timestamp,{self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def arm_config(wl: "Workload", world: int) -> dict:
    """The `config` object of a bench line -- the same for our arm and for --impl reference
    (the reference arm runs on our arm's config): built from the workload and the rank count
    alone, rank 0's share standing for the per-GPU figures."""
    B = len(wl.local_specs(0, world))
    px = B * wl.W * wl.H
    return {"workload": wl.desc + ", fg8_bg4, features+Euler+tree+hole fill",
            "images_per_gpu": B, "pixels_per_gpu": px,
            "l2": "inputs > L2 (no flush)" if px > 126e6 else "inputs fit L2 (cfg1/cfg3 are launch-bound single images)",
            "pipelines": PIPELINES,
            "parallelism": (f"batch sharded by image x{world} (cost-balanced, no data-path "
                            "collective)" if wl.shard and world > 1
                            else f"replica per rank x{world}")}


# ------------------------------------------------------------------------------ CPU side
def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def time_reference(imgs: np.ndarray, threads: int) -> float:
    from oracle import oracle as O
    secs, _ = O.ref_time_batch(imgs, 0, threads)
    return secs


def run_reference_arm(args, wl: Workload, rank: int) -> None:
    """--impl reference: the reference's own CPU path, all host threads, rank 0 only."""
    if rank != 0:
        return
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libref_runlab.so not built"}))
        return
    threads = cpu_threads()
    specs = wl.specs if wl.name != "cfg4" else wl.specs[:512]
    imgs = wl.make_host(specs)
    px = imgs.shape[0] * wl.W * wl.H
    for _ in range(args.warmup):
        time_reference(imgs, threads)
    times = [time_reference(imgs, threads) for _ in range(args.steps)]
    t = sum(times) / len(times)
    value = px / t / 1e9
    sample = (f"{imgs.shape[0]} images of {wl.W}x{wl.H} per step"
              + (" (first 512 of 4096)" if wl.name == "cfg4" else " (the full workload)")
              + ", one image per thread")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gpixel/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong" if (wl.shard and args.gpus > 1) else "weak",
        "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (reference generator)",
        "config": arm_config(wl, max(1, args.gpus)),
        "reference_path": "label_image(features,euler) + label_image(fill,features,relabel) + binarize_labels",
        "cpu_baseline": {"value": value, "unit": "Gpixel/s", "cores": threads, "kind": "reference",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def _compare_image(got: dict, ref) -> str | None:
    """None when one image's GPU outputs equal the reference's canonical result bit for bit,
    else the first differing field (SURVEY 8(d) parity list)."""
    for k in ("n_components", "n_fg", "n_holes", "euler", "n_survivors"):
        if got[k] != getattr(ref, k):
            return k
    if got["comps"].tobytes() != ref.comps.tobytes():
        return "comps"
    if not np.array_equal(got["top"], ref.top):
        return "top"
    surv = ref.top == np.arange(ref.n_components, dtype=np.uint32)
    if got["filled"][surv].tobytes() != ref.filled[surv].tobytes():
        return "filled"
    if not np.array_equal(got["filled_image"], ref.filled_image):
        return "filled_image"
    return None


def parity_check(wl: Workload, specs, res, threads: int) -> dict:
    """Every image of the timed batch against the reference compiled from its own headers
    (oracle/_ref; the C restatement when it is absent), outside the timed region.  Images are
    generated on the host with the oracle's generator, labeled by the reference and compared
    with `res` (the fetched device result) by a pool of host threads (the ctypes calls release
    the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O
    use_ref = O.ref_available()
    label = O.ref_label_canonical if use_ref else O.label_canonical
    t0 = time.perf_counter()

    def one(i: int):
        s = specs[i]
        img = (O.generate(wl.W, wl.H, s[1], s[2], s[3]) if s[0] == "gen"
               else O.generate_rings(wl.W, wl.H, s[1], s[2], s[3]))
        return _compare_image(res.image(i), label(img, 0))

    with ThreadPoolExecutor(max(1, threads)) as ex:
        bad = [(i, f) for i, f in enumerate(ex.map(one, range(len(specs)))) if f is not None]
    n = len(specs)
    return {"images": n, "mismatches": len(bad), "first_mismatch": bad[:3] or None,
            "against": "reference (oracle/_ref)" if use_ref else "C restatement (oracle/liboracle.so)",
            "summary": (f"bit-exact {n - len(bad)}/{n}" if not bad else f"MISMATCH {len(bad)}/{n}"),
            "seconds": time.perf_counter() - t0}


def relaunch_distributed(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: run this script under torch.distributed.run with
    N ranks on this node (the driver's own launch line), NCCL_DEBUG=INFO into a log file."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_FILE", os.path.join("/tmp", "runlab_bench_nccl.%h.%p.log"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------------------------ our arm
def run_strips(args, wl: Workload, rank: int, world: int, local: int) -> None:
    """the single image of the workload cut into one horizontal strip per rank;
    four collectives per step, O(width) bytes each (strips.py).  Strong scaling: the image is
    fixed."""
    import torch
    import torch.distributed as dist

    from paper_2006_09299_b200 import Labeler, LabelingConfig
    from paper_2006_09299_b200.runlab import generate_rows_device
    from paper_2006_09299_b200.strips import HostStagedCollectives, TorchCollectives, label_strip, strip_rows

    if len(wl.specs) != 1 or wl.specs[0][0] != "gen":
        raise SystemExit("--strips needs a single generated image (cfg1 or cfg5)")
    torch.cuda.set_device(local)
    dist.init_process_group(BACKEND, device_id=torch.device("cuda", local) if BACKEND == "nccl" else None)
    y0, h = strip_rows(wl.H, world)[rank]
    _, dens, gran, seed = wl.specs[0]
    d = torch.empty((h, wl.W), dtype=torch.uint8, device="cuda")
    generate_rows_device(d.data_ptr(), wl.W, wl.H, y0, h, dens, gran, seed)
    torch.cuda.synchronize()
    lab = Labeler(local)
    coll = TorchCollectives() if BACKEND == "nccl" else HostStagedCollectives()
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    stream = torch.cuda.ExternalStream(lab.stream())

    def step(fetch=False):
        return label_strip(lab, d.data_ptr(), wl.W, wl.H, y0, h, cfg, coll, fetch=fetch)

    for _ in range(args.warmup):
        res = step()
    clocks = ClockSampler(local)
    clocks.start()
    t_busy = time.time() + 0.3  # the GPU is under load before the timed region
    while time.time() < t_busy:
        step()
    dist.barrier()
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = step()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    launches = lab.launch_count() * args.steps
    t_busy = time.time() + 0.3
    while time.time() < t_busy:
        step()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms_step = statistics.mean(times)
    t = torch.tensor([ms_step], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item())
    P = wl.W * wl.H
    # e2e: host strip in, owned outputs out (pinned), through the same phases
    h_in = torch.empty((h, wl.W), dtype=torch.uint8, pin_memory=True)
    h_in.copy_(d.cpu())
    dist.barrier()
    full = step(fetch=True)  # allocates the pinned staging buffers once
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(max(args.e2e_steps, 1)):
        d.copy_(h_in, non_blocking=True)
        torch.cuda.synchronize()
        full = step(fetch=True)
    e2e_s = (time.perf_counter() - t0) / max(args.e2e_steps, 1)
    t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    owned = full.comp_hi - full.comp_lo
    c_pre, c_post = res.n_components, res.n_survivors
    bytes_alg = 2 * P + 48 * c_pre + 40 * c_post
    peak, peak_src = measured_peaks()
    per_gpu_gbs = bytes_alg / world / (ms_step / 1e3) / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": P / (ms_step / 1e3) / 1e9, "unit": "Gpixel/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (reference generator on device, each rank generates its own rows)",
            "config": {"workload": wl.desc + ", fg8_bg4, features+Euler+tree+hole fill",
                       "images_per_gpu": 1.0 / world, "pixels_per_gpu": P // world,
                       "l2": "inputs > L2 (no flush)" if P // world > 126e6 else "strip fits L2",
                       "parallelism": f"horizontal strips x{world} (all-gather of cut-class tables and "
                                      "cut-row labels, all-reduce of cut components' links and of "
                                      "cut survivors' partial features)"},
            "roofline": {"bound": "hbm", "kernel": "whole strip step (per GPU)", "achieved": per_gpu_gbs,
                         "peak": peak, "unit": "GB/s", "frac": per_gpu_gbs / peak, "traffic": None,
                         "peak_source": peak_src, "c_pre": c_pre, "c_post": c_post},
            "cpu_baseline": None,
            "e2e": {"value": P / e2e_s / 1e9, "unit": "Gpixel/s", "h2d_bytes_per_step": h * wl.W,
                    "d2h_bytes_per_step": h * wl.W + 92 * owned, "ms_per_step": e2e_s * 1e3,
                    "api": "strips.label_strip (pinned host strip in, owned components + strip of the "
                           "filled image out)"},
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line))
    lab.close()
    dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the bit-exact check against the reference")
    ap.add_argument("--cpu-seconds", type=float, default=5.0, help="minimum timed wall time of the CPU baseline")
    ap.add_argument("--strips", action="store_true",
                    help="one image cut into horizontal strips across the ranks (default for cfg5 with N > 1)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        raise SystemExit(relaunch_distributed(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # testing aid for the N > 1 code path on a one-GPU box: every rank on GPU 0 over gloo
    # (RUNLAB_BENCH_SHARED_GPU=1); never set by the driver
    global BACKEND
    if os.environ.get("RUNLAB_BENCH_SHARED_GPU"):
        local, BACKEND = 0, "gloo"
    wl = Workload(args.config)

    if args.impl == "reference":
        run_reference_arm(args, wl, rank)
        return
    args.warmup = max(args.warmup, 3)
    if args.strips or (wl.name == "cfg5" and world > 1):
        run_strips(args, wl, rank, world, local)
        return

    import torch
    import torch.distributed as dist

    from paper_2006_09299_b200 import Labeler, LabelingConfig
    from paper_2006_09299_b200 import _native as N
    from paper_2006_09299_b200.distributed import sum_over_ranks

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group(BACKEND, device_id=torch.device("cuda", local) if BACKEND == "nccl" else None)

    specs = wl.local_specs(rank, world)
    B = len(specs)
    P = wl.W * wl.H
    imgs = wl.make_device(specs)

    lab = Labeler(local)
    lab.set_pipelines(PIPELINES)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    stream = torch.cuda.ExternalStream(lab.stream())

    def step():
        lab.label_device(imgs.data_ptr(), wl.W, wl.H, B, cfg)

    for _ in range(args.warmup):
        step()
        lab.sync()  # settles capacity estimates before timing

    clocks = ClockSampler(local)
    clocks.start()
    t_busy = time.time() + 0.3  # the GPU is under load before the timed region
    while time.time() < t_busy:
        step()
        lab.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    lab.sync()  # raises if the device flagged an error
    ms = ev0.elapsed_time(ev1)
    launches_per_step = lab.launch_count()
    res = lab.fetch()  # the timed calls' outputs (parity below checks every image of them)
    if world > 1:
        dist.barrier()
    t_busy = time.time() + 0.3  # same load a little longer: the sampler brackets the region
    while time.time() < t_busy:
        step()
        lab.sync()
    clk = clocks.stop()
    # per-phase device times (library events on its stream) for the roofline: a large batch
    # runs as concurrent pipelines whose phases overlap, so the phases are timed on the same
    # batch run as one pipeline (untimed for the value)
    lab.set_pipelines(1)
    for _ in range(3):
        step()
        lab.sync()
    nph = 5
    for _ in range(nph):
        step()
    lab.sync()
    phases = ([lab.phase_times(0)] if lab.used_graph()
              else [lab.phase_times(k) for k in range(nph)])
    one_pipeline_ms = statistics.mean(p.total_ms for p in phases)
    lab.set_pipelines(PIPELINES)

    ms_step = ms / args.steps
    if world > 1:
        t = torch.tensor([ms_step], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    ana = statistics.mean(p.analyze_ms for p in phases)
    mer = statistics.mean(p.merge_ms for p in phases)
    emi = statistics.mean(p.emit_ms for p in phases)

    # component counts for the algorithmic byte count
    c_pre = int(res.n_components.sum())
    c_post = int(res.n_survivors.sum())
    px = B * P
    total_px = px
    if world > 1:
        t = torch.tensor([px], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        total_px = int(t.item())
    bytes_alg = 2 * px + 48 * c_pre + 40 * c_post
    peak, peak_src = measured_peaks()
    pipe_gbs = bytes_alg / (ms_step / 1e3) / 1e9
    dom = max((("k_analyze", ana, px), ("k_emit", emi, px + 48 * c_pre + 40 * c_post)), key=lambda x: x[1])
    dom_gbs = dom[2] / (dom[1] / 1e3) / 1e9
    traffic, traffic_src = profiled_traffic(args.config, dom[0])

    # ---- e2e: the host-buffer C-ABI call (pinned host in/out, copies inside the timed region)
    e2e = None
    if args.e2e_steps > 0:
        h_in = torch.empty((B, wl.H, wl.W), dtype=torch.uint8, pin_memory=True)
        h_in.copy_(imgs.cpu())
        h_fill = torch.empty((B, wl.H, wl.W), dtype=torch.uint8, pin_memory=True)
        cap = c_pre + 1024
        h_comps = torch.empty(cap * 48, dtype=torch.uint8, pin_memory=True)
        h_top = torch.empty(cap * 4, dtype=torch.uint8, pin_memory=True)
        h_filled = torch.empty((c_post + 1024) * 40, dtype=torch.uint8, pin_memory=True)
        h_summ = torch.empty(B * 5, dtype=torch.int64, pin_memory=True)
        h_off = torch.empty(B + 1, dtype=torch.int64, pin_memory=True)
        outs = N.RlHostOutputs(h_fill.data_ptr(), None, h_comps.data_ptr(), h_top.data_ptr(),
                               h_filled.data_ptr(), cap, h_summ.data_ptr(), h_off.data_ptr(), 0, 0, 0,
                               1, 0)  # post-fill features of the survivors only
        lab.label_into(h_in.data_ptr(), wl.W, wl.H, B, cfg, outs)  # warm
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            lab.label_into(h_in.data_ptr(), wl.W, wl.H, B, cfg, outs)
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        assert np.array_equal(h_summ.numpy().reshape(B, 5)[:, 0], res.n_components), "e2e result mismatch"
        e2e = {"value": total_px / e2e_s / 1e9, "unit": "Gpixel/s",
               "h2d_bytes_per_step": int(outs.h2d_bytes), "d2h_bytes_per_step": int(outs.d2h_bytes),
               "ms_per_step": e2e_s * 1e3,
               "api": "rl_label_into (pinned host pixels in; filled image, component records, "
                      "post-fill roots, survivors' post-fill features, per-image counts out; "
                      "chunks of whole images pipelined over 3 streams)"}
        # the same call with PBM P4 rasters in and out (1 bit per pixel over PCIe, the
        # reference CLI's file format): reported beside, not as the headline
        from paper_2006_09299_b200.runlab import pack_p4
        h_p4 = torch.from_numpy(pack_p4(h_in.numpy())).pin_memory()
        h_fp4 = torch.empty_like(h_p4).pin_memory()
        outs4 = N.RlHostOutputs(h_fp4.data_ptr(), None, h_comps.data_ptr(), h_top.data_ptr(),
                                h_filled.data_ptr(), cap, h_summ.data_ptr(), h_off.data_ptr(), 0, 0, 0, 1, 0)
        lab.label_into(h_p4.data_ptr(), wl.W, wl.H, B, cfg, outs4, pixel_format=N.RL_PIXELS_P4)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            lab.label_into(h_p4.data_ptr(), wl.W, wl.H, B, cfg, outs4, pixel_format=N.RL_PIXELS_P4)
        p4_s = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([p4_s], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            p4_s = float(t.item())
        assert np.array_equal(h_summ.numpy().reshape(B, 5)[:, 0], res.n_components), "e2e P4 result mismatch"
        e2e["p4"] = {"value": total_px / p4_s / 1e9, "unit": "Gpixel/s", "ms_per_step": p4_s * 1e3,
                     "h2d_bytes_per_step": int(outs4.h2d_bytes), "d2h_bytes_per_step": int(outs4.d2h_bytes),
                     "api": "rl_label_into_fmt(RL_PIXELS_P4): P4 rows in, filled image as P4 rows out"}

    # ---- parity of the timed batch (every image, every output) against the reference
    parity = None
    if not args.no_parity:
        parity = parity_check(wl, specs, res, max(1, cpu_threads() // world))
        if world > 1:
            bad = sum_over_ranks(parity["mismatches"], device="cuda")
            tot = sum_over_ranks(parity["images"], device="cuda")
            parity["images"], parity["mismatches"] = tot, bad
            parity["summary"] = f"bit-exact {tot - bad}/{tot}" if not bad else f"MISMATCH {bad}/{tot}"

    # ---- CPU baseline: the reference itself on a bounded sample, rank 0 at N=1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import oracle as O
            sample_specs, sample_desc = wl.cpu_sample()
            if O.ref_available() and sample_specs is not None:
                h_imgs = wl.make_host(sample_specs)
                threads = cpu_threads()
                time_reference(h_imgs, threads)  # warm-up pass
                secs, passes = 0.0, 0
                while secs < args.cpu_seconds or passes == 0:
                    secs += time_reference(h_imgs, threads)
                    passes += 1
                cpu = {"value": passes * h_imgs.shape[0] * P / secs / 1e9, "unit": "Gpixel/s", "cores": threads,
                       "kind": "reference",
                       "sample": f"{sample_desc} x {passes} timed passes after one warm-up pass, one image "
                                 "per thread, same-outputs path (2x label_image + binarize_labels)",
                       "cpu": cpu_model(), "seconds": secs}
            elif sample_specs is None:
                cpu = {"value": None, "unit": "Gpixel/s", "cores": 0, "kind": "reference", "sample": sample_desc}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "Gpixel/s", "cores": 0, "kind": "reference",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        scaling = "strong" if (wl.shard and world > 1) else "weak"
        line = {
            "metric": METRIC, "value": total_px / (ms_step / 1e3) / 1e9, "unit": "Gpixel/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (reference generator on device)",
            "config": arm_config(wl, world),
            "parity": parity,
            "roofline": {"bound": "hbm", "kernel": dom[0] + " (+ deferred-class launches)", "achieved": dom_gbs,
                         "peak": peak, "unit": "GB/s", "frac": dom_gbs / peak, "traffic": traffic,
                         "traffic_source": traffic_src, "peak_source": peak_src,
                         "alg_bytes_per_launch": dom[2], "avg_launch_ms": dom[1],
                         "pipeline": {"alg_bytes_per_step": bytes_alg, "achieved": pipe_gbs,
                                      "frac": pipe_gbs / peak, "c_pre": c_pre, "c_post": c_post,
                                      "phase_ms": {"analyze": ana, "merge": mer, "emit": emi},
                                      "phase_source": "CUDA events of the same batch run as one pipeline "
                                                      f"({one_pipeline_ms:.4f} ms per step; the timed "
                                                      "calls overlap their pipelines' phases)"}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
        }
        print(json.dumps(line))
    lab.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
