"""Benchmark: 3D hull points/sec on the B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4]
                    [--impl ours|reference] [--engine fast|exact]

One "step" = one full ``convex_hull_3d`` of the config's point cloud: device
presort + tie scan + degeneracy scan, both hull passes over all merge
levels, facet extraction and the orientation/remap/unique epilogue.

* ``value``: points/sec with the input cloud already resident in HBM (caller
  order, 24 B/point; 2^24 points = 403 MB > the 126 MB L2, so every step
  streams it from HBM), device events around K steps.
* ``e2e``: the same metric through the public API with HOST buffers: every
  step copies the pinned input host->device and reads faces + vertices back.
* ``roofline``: the dominant kernel's algorithmic bytes (SURVEY.md 8(d)
  model, per-level counts frozen from the reference in
  tests/golden/level_stats.json) over its event-timed launch durations,
  against MEASURED_PEAKS.json hbm_gbs.
* ``cpu_baseline``: the unmodified reference (oracle/_ref) on this host's
  cores on a bounded sample, rank 0 only.

``--impl reference`` times the reference's own CPU implementation
(ThreadBackend over all host cores) on a bounded sample of the same
workload and prints the same JSON line with "impl": "reference".
Multi-GPU (torchrun, N>1): x-slab sharding, see DESIGN.md.
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

CONFIGS = {
    # name: (n, dist, seed, label)
    "C1": (10_000, "cube", 0, "10^4 uniform cube [-1,1]^3"),
    "C2": (2**20, "ball", 0, "2^20 uniform unit ball"),
    "C3": (2**20, "sphere", 0, "2^20 sphere surface (h~n)"),
    "C4": (2**24, "cube", 0, "2^24 uniform cube [-1,1]^3"),
    "C5": (2**27, "mixed", 0, "2^27 ball + 2^20 radius-2 shell"),
    # BASELINE.md "Integer" row: integer coordinates in [-2^30, 2^30) (tie path)
    "INT": (2**20, "int31", 0, "2^20 integer cloud, coordinates in [-2^30, 2^30)"),
}
# full-size CPU runs per config (the reference at C5 takes ~140 s per call on
# 8 threads: the only config whose CPU legs run a bounded sample)
CPU_FULL_MAX = 2**24


def make_points(cfg: str) -> np.ndarray:
    from paper_1205_1171_b200.generators import generate, integer_cloud

    n, dist, seed, _ = CONFIGS[cfg]
    if dist == "int31":
        return integer_cloud(n, seed)
    return generate(n, dist, seed)


def sample_points(cfg: str, sn: int) -> np.ndarray:
    from paper_1205_1171_b200.generators import generate, integer_cloud

    n, dist, seed, _ = CONFIGS[cfg]
    if sn >= n:
        return make_points(cfg)
    if dist == "int31":
        return integer_cloud(sn, seed)
    return generate(sn, dist, seed)
STATS_KEY = {"C2": "C2_ball_2^20", "C3": "C3_sphere_2^20", "C4": "C4_cube_2^24",
             "INT": "int_2^20_R2^31", "C5": "C5_mixed_2^27"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--engine", default="fast", choices=["fast", "exact"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-n", type=int, default=CPU_FULL_MAX,
                    help="largest cloud the CPU legs run (configs above it use a sample)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, flag in zip(names, parts[5:9]):
                if flag.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# -------------------------------------------------------------- reference
def reference_module():
    from oracle import oracle as O

    ref = O.reference()
    if ref is None:
        raise RuntimeError("reference not built: run oracle/build_ref.sh (or __graft_entry__.build())")
    return ref


def time_reference(pts: np.ndarray, reps: int, warm: int = 1, serial: bool = False):
    """Reference convex_hull_3d on ``pts``: ThreadBackend(all host cores), or
    the 1-core top-down ``solver="serial"``.  Returns (seconds list, cores)."""
    ref = reference_module()
    if serial:
        out = []
        for i in range(warm + reps):
            t0 = time.perf_counter()
            ref.convex_hull_3d(pts, solver="serial")
            dt = time.perf_counter() - t0
            if i >= warm:
                out.append(dt)
        return out, 1
    cores = os.cpu_count() or 1
    out = []
    with ref.ThreadBackend(cores) as be:
        for i in range(warm + reps):
            t0 = time.perf_counter()
            ref.convex_hull_3d(pts, be)
            dt = time.perf_counter() - t0
            if i >= warm:
                out.append(dt)
    return out, cores


def cpu_baseline(cfg: str, sample_n: int) -> dict:
    """The unmodified reference on this host (rank 0, N=1 only): the whole
    config cloud (up to ``sample_n`` points), one timed call of the leveled
    solver on every host core and one of the 1-core serial solver (the two
    CPU numbers BASELINE.md 2 asks for), no warm-up (a call is seconds long)."""
    n, dist, seed, _ = CONFIGS[cfg]
    sn = min(n, sample_n)
    pts = sample_points(cfg, sn)
    what = "the full config cloud" if sn == n else f"a bounded sample of {cfg}"
    secs, cores = time_reference(pts, reps=1, warm=0)
    ser, _ = time_reference(pts, reps=1, warm=0, serial=True)
    return {"value": sn / secs[0], "unit": "points/s", "cores": cores, "kind": "reference",
            "sample": f"reference convex_hull_3d(ThreadBackend({cores})) on {sn} points "
                      f"({what}: {cfg} n={n}, dist {dist!r}, seed {seed}), 1 timed call, "
                      f"no warm-up; host CPU {cpu_model()}",
            "seconds": secs[0],
            "serial_1core": {"value": sn / ser[0], "unit": "points/s", "cores": 1,
                             "seconds": ser[0],
                             "sample": f"reference convex_hull_3d(solver='serial') on the "
                                       f"same {sn} points, 1 timed call"}}


def run_reference_arm(args):
    """The reference's own CPU implementation (unmodified, oracle/_ref) on
    this host: ThreadBackend over all host cores, every step one full
    convex_hull_3d of the config cloud (C5, 2^27, runs a 2^24 sample).
    Rank 0 only; other ranks exit without work."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    n, dist, seed, label = CONFIGS[args.config]
    sn = min(n, args.cpu_sample_n)
    pts = sample_points(args.config, sn)
    secs, cores = time_reference(pts, reps=args.steps, warm=args.warmup)
    total = sum(secs)
    value = sn * len(secs) / total
    cfg = {"workload": f"{args.config}: {label}", "n": n, "distribution": dist, "seed": seed}
    if sn != n:
        cfg["sample_n"] = sn
    what = "the full config cloud" if sn == n else f"a {sn}-point sample"
    line = {
        "impl": "reference", "metric": "3D hull points/sec", "value": value, "unit": "points/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / len(secs) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator, PCG64)",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "reference",
                         "sample": f"{what} per step ({args.steps} timed after {args.warmup} "
                                   f"warm-up); host CPU {cpu_model()}"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- ours
def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def level_stats(cfg: str):
    key = STATS_KEY.get(cfg)
    p = os.path.join(ROOT, "tests", "golden", "level_stats.json")
    if key is None or not os.path.exists(p):
        return None
    return json.load(open(p)).get(key)


def level_bytes(cfg: str):
    """Algorithmic bytes per (pass, level) row of the profile:
    a per-level merge is credited B_alg = 4(E_in+E_out) + 40(D+2J); the fused
    leaf kernel (profile level -b = levels 1..b in one launch) is credited
    once: 4*E_in(1) + 4*E_out(b) + 40*(points in its groups) -- one 32-byte
    record read + one 8-byte link write per point -- not the per-level sum."""
    st = level_stats(cfg)
    if st is None:
        return None
    n = CONFIGS[cfg][0]
    out = {}
    for pi, which in enumerate(("lower", "upper")):
        rows = {r["level"]: r for r in st[which]}
        for lv, r in rows.items():
            out[(pi, lv)] = 4 * (r["E_in"] + r["E_out"]) + 40 * (r["D"] + 2 * r["J"])
            out[(pi, -lv)] = 4 * rows[1]["E_in"] + 4 * r["E_out"] + 40 * n
    # pass index 2: one launch covering both passes of a level
    for (pi, lv), b in list(out.items()):
        if pi == 0 and (1, lv) in out:
            out[(2, lv)] = b + out[(1, lv)]
    return out


# bench kernel names -> the ncu kernel names they cover
NCU_NAMES = {
    # the lane-per-job route: lane.cu (levels <= 5) and k_fast_tpj above
    "k_fast_tpj": ("h3d::k_fast_tpj<", "h3d::k_fast_tpj_r128<", "h3d::k_lane<"),
    "k_fast_warp": ("h3d::k_fast_warp<",),
    "k_fast_leaf": ("h3d::k_fast_leaf<",),
    "k_fast_init1": ("h3d::k_fast_init1",),
    "k_big_level": ("h3d::k_big_",),
    "k_mini": ("h3d::k_mini<",),
}


def measured_inst(cfg: str, name: str):
    """Warp instructions per launch (smsp__inst_executed.sum) of the kernel,
    from the same committed ncu launch list as measured_traffic."""
    import glob

    cands = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_ncu_launches_{cfg.lower()}.json")),
                   key=lambda q: int(os.path.basename(q)[1:].split("_", 1)[0]))
    if not cands:
        return None
    doc = json.load(open(cands[-1]))
    pre = NCU_NAMES.get(name, (name,))
    ks = [k for k in doc["kernels"] if k["kernel"].startswith(pre) and k.get("warp_inst")]
    if not ks or name == "k_big_level":
        return None
    return sum(k["warp_inst"] for k in ks) // max(sum(k["launches"] for k in ks), 1)


def measured_traffic(cfg: str, name: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
    of the kernel, from the committed ncu launch list of this config
    (profiles/r<round>_ncu_launches_<cfg>.json, the latest round's, made by tools/evidence_r2.sh +
    tools/ncu_summary.py).  A big-level "launch" is the pipeline's kernels of
    one level; it is counted per level."""
    import glob

    cands = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_ncu_launches_{cfg.lower()}.json")),
                   key=lambda q: int(os.path.basename(q)[1:].split("_", 1)[0]))
    if not cands:
        return None, None
    p = cands[-1]  # the latest round's launch list
    doc = json.load(open(p))
    pre = NCU_NAMES.get(name, (name,))
    ks = [k for k in doc["kernels"] if k["kernel"].startswith(pre)]
    if not ks:
        return None, None
    total = sum(k["dram_bytes"] for k in ks)
    if name == "k_big_level":
        levels = sum(1 for x in doc["sequence"] if x["kernel"] == "h3d::k_big_jobs")
        per = total // max(levels, 1)
    else:
        per = total // max(sum(k["launches"] for k in ks), 1)
    return per, os.path.relpath(p, ROOT)


def run_ours(args):
    import torch

    import paper_1205_1171_b200 as H
    from paper_1205_1171_b200 import engine as E

    ws, rank, local = dist_env()
    if ws > 1:
        return run_ours_distributed(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n, dist, seed, label = CONFIGS[args.config]
    pts_host = make_points(args.config)
    pinned = torch.from_numpy(pts_host).pin_memory()
    pts_dev = pinned.to(dev)
    be = H.CudaBackend(local, engine=args.engine)
    from paper_1205_1171_b200 import fast as F
    fb0 = F.FALLBACKS[0]
    stream = torch.cuda.current_stream(dev)

    for _ in range(max(args.warmup, 3)):
        res = H.convex_hull_3d(pts_dev, be, return_device=True)
    torch.cuda.synchronize()
    nfaces = int(res.faces.shape[0])
    nverts = int(res.vertices.shape[0])

    # device-resident timed region: per-level times come from the level
    # kernels' own device time stamps (no event records); CUDA events bracket
    # only the lane-per-job kernel launches (the dominant kernel: roofline)
    prof: list = []
    E.KERNEL_EVENTS = True
    F.profile_collect(1 << 20)  # drop the warm-up's records
    l0 = E.launch_count()
    y0 = E.sync_count()
    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        H.convex_hull_3d(pts_dev, be, return_device=True)
    ev1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    for tag, p_idx, t_ms in F.profile_collect(1 << 20):
        name, lv = F.kernel_of(tag)
        prof.append((name, p_idx, lv, t_ms))
    E.KERNEL_EVENTS = False
    launches = (E.launch_count() - l0) // args.steps
    host_syncs = (E.sync_count() - y0) / args.steps
    ms = ev0.elapsed_time(ev1) / args.steps
    value = n / (ms / 1e3)
    fallbacks = F.FALLBACKS[0] - fb0
    # which route each level took in the last timed step (fused fast path
    # vs exact engine), from the device level stamps
    routes: dict = {}
    level_ms: dict = {}
    for tag, _p, t_ms in F.LAST_LEVEL_ROWS:
        name, lv = F.kernel_of(tag)
        routes[name] = routes.get(name, 0) + 1
        level_ms[str(lv)] = round(t_ms, 4)
    routes = dict(sorted(routes.items()))
    # the presort, reported separately: 68 algorithmic
    # bytes per point (8 B key read + 4 B permutation write + 24 B row
    # gather + 32 B record write), over its device time in the last step
    presort = None
    if F.LAST_SORT_MS[0]:
        pb = 68 * n
        pms = F.LAST_SORT_MS[0]
        presort = {"ms": pms, "bytes_alg": pb, "achieved_gbps": pb / pms / 1e6,
                   "frac": pb / pms / 1e6 / peak_hbm()[0], "share_of_step": pms / ms}

    # roofline of the dominant kernel
    per_kernel: dict = {}
    lb = level_bytes(args.config)
    for name, pass_idx, level, t_ms in prof:
        t = t_ms / 1e3
        d = per_kernel.setdefault(name, {"time": 0.0, "launches": 0, "bytes": 0, "known": True})
        d["time"] += t
        d["launches"] += 1
        b = None if lb is None else lb.get((pass_idx, level))
        if b is None:
            d["known"] = False
        else:
            d["bytes"] += b
    peak, peak_kind = peak_hbm()
    roof = None
    if per_kernel:
        name, d = max(per_kernel.items(), key=lambda kv: kv[1]["time"])
        ach = d["bytes"] / d["time"] / 1e9 if d["known"] and d["time"] > 0 else None
        nl = max(d["launches"], 1)
        traffic, tsrc = measured_traffic(args.config, name)
        label = "lane-per-job (k_lane, k_fast_tpj)" if name == "k_fast_tpj" else name
        roof = {"bound": "hbm", "kernel": label, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": (ach / peak) if ach else None,
                "traffic": traffic,
                "traffic_source": tsrc,
                "algorithmic_bytes_per_launch": d["bytes"] // nl,
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                "launches_per_step": d["launches"] // args.steps,
                "kernel_ms_per_step": d["time"] * 1e3 / args.steps,
                "share_of_step": d["time"] * 1e3 / args.steps / ms,
                "bytes_per_step": d["bytes"] // args.steps}
        # the bound these sweeps actually meet: instruction issue (4 warp
        # instructions per SM per cycle at the measured SM clock), from the
        # ncu instruction count per launch and this run's kernel time
        wi = measured_inst(args.config, name)
        if wi and d["time"] > 0:
            sm_mhz = (clk or {}).get("sm_mhz") or 1965.0
            peak_issue = 4 * torch.cuda.get_device_properties(dev).multi_processor_count * sm_mhz * 1e6
            got = wi * d["launches"] / d["time"]
            roof["issue"] = {"achieved": got, "peak": peak_issue, "unit": "warp instructions/s",
                             "frac": got / peak_issue, "warp_inst_per_launch": wi,
                             "source": "smsp__inst_executed.sum, " + (tsrc or "")}

    # end to end through the public API with host buffers (W untimed calls
    # first: the pinned result buffers come from torch's caching host
    # allocator; keeping each result alive until the next call returns, as
    # the timed loop does, caches both generations of buffers)
    r = None
    for _ in range(max(args.warmup, 2)):
        r = H.convex_hull_3d(pinned, be)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        r = H.convex_hull_3d(pinned, be)
    ev1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = ev0.elapsed_time(ev1) / args.steps
    e2e = {"value": n / (e2e_ms / 1e3), "unit": "points/s", "h2d_bytes_per_step": 24 * n,
           "d2h_bytes_per_step": int(r.faces.nbytes + r.vertices.nbytes), "ms_per_step": e2e_ms,
           "api": "convex_hull_3d(pinned host cloud) -> numpy faces/vertices, one call per step"}
    # the same through the streaming extension: step i+1's host->device copy
    # overlaps step i's hull (every step still copies its whole cloud and
    # reads its result back)
    for _ in H.convex_hull_3d_stream([pinned] * max(args.warmup, 2), be):
        pass
    torch.cuda.synchronize()
    ev0.record(stream)
    rs = 0
    for r in H.convex_hull_3d_stream([pinned] * args.steps, be):
        rs += int(r.faces.shape[0])
    ev1.record(stream)
    torch.cuda.synchronize()
    pe_ms = ev0.elapsed_time(ev1) / args.steps
    e2e_pipelined = {"value": n / (pe_ms / 1e3), "unit": "points/s", "h2d_bytes_per_step": 24 * n,
                     "d2h_bytes_per_step": int(r.faces.nbytes + r.vertices.nbytes),
                     "ms_per_step": pe_ms,
                     "api": "convex_hull_3d_stream (copy of cloud i+1 on a second stream during hull i)"}

    cpu = None
    if not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.config, args.cpu_sample_n)
        except Exception as exc:  # reference missing on this box
            cpu = {"value": None, "unit": "points/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    line = {
        "metric": "3D hull points/sec", "value": value, "unit": "points/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, PCG64)",
        "config": {"workload": f"{args.config}: {label}", "n": n, "distribution": dist,
                   "seed": seed, "engine": args.engine, "parallelism": "1 GPU",
                   "l2": "input 24n bytes > 126 MB L2 (C4/C5); no explicit flush",
                   "faces": nfaces, "vertices": nverts},
        "e2e": e2e, "e2e_pipelined": e2e_pipelined, "gpu_launches": launches,
        "host_syncs_per_step": host_syncs, "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk, "fallbacks": fallbacks, "routes_per_step": routes,
        "level_ms_last_step": level_ms,
        "presort": presort,
    }
    print(json.dumps(line), flush=True)


def run_ours_distributed(args):
    """N ranks (torchrun): x-slab sharding with NCCL point-to-point for the
    final log2 G levels (paper_1205_1171_b200/multigpu.py).  Every rank holds
    the input; the time is the max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1205_1171_b200 import engine as E
    from paper_1205_1171_b200.multigpu import SlabPlan, convex_hull_3d_distributed

    ws, rank, local = dist_env()
    if os.environ.get("H3D_DIST_ONE_GPU"):
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # H3D_DIST_BACKEND=gloo (+ H3D_DIST_ONE_GPU=1): a functional run of this
    # multi-rank path on a one-GPU box (timings meaningless); NCCL otherwise
    if os.environ.get("H3D_DIST_BACKEND", "nccl") == "gloo":
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    n, dist_name, seed, label = CONFIGS[args.config]
    pts_host = make_points(args.config)
    pinned = torch.from_numpy(pts_host).pin_memory()
    pts_dev = pinned.to(dev)
    stream = torch.cuda.current_stream(dev)

    def timed(fn):
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = None
        for _ in range(args.steps):
            out = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), out

    for _ in range(max(args.warmup, 3)):
        convex_hull_3d_distributed(pts_dev, dev, return_device=True)
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    l0 = E.launch_count()
    ms, res = timed(lambda: convex_hull_3d_distributed(pts_dev, dev, return_device=True))
    launches = (E.launch_count() - l0) // args.steps
    clk = clocks.stop() if clocks else None
    r = None
    for _ in range(max(args.warmup, 2)):
        r = convex_hull_3d_distributed(pinned, dev)  # kept alive: see the 1-GPU path
    e2e_ms, r = timed(lambda: convex_hull_3d_distributed(pinned, dev))
    # one untimed call with phase events: where a rank's step goes
    import paper_1205_1171_b200.multigpu as MG
    MG.PHASES = []
    convex_hull_3d_distributed(pts_dev, dev, return_device=True)
    phases = MG.PHASES[0] if MG.PHASES else None
    MG.PHASES = None
    if rank != 0:
        dist.destroy_process_group()
        return
    plan = SlabPlan(n, ws)
    line = {
        "metric": "3D hull points/sec", "value": n / (ms / 1e3), "unit": "points/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, PCG64)",
        "config": {"workload": f"{args.config}: {label}", "n": n, "distribution": dist_name,
                   "seed": seed, "engine": "fast", "parallelism": f"x-slab x{plan.G}",
                   "slab_level": plan.slab_level,
                   "l2": "input 24n bytes > 126 MB L2 (C4/C5); no explicit flush",
                   "faces": int(res.faces.shape[0]), "vertices": int(res.vertices.shape[0])},
        "e2e": {"value": n / (e2e_ms / 1e3), "unit": "points/s", "h2d_bytes_per_step": 24 * n,
                "d2h_bytes_per_step": int(r.faces.nbytes + r.vertices.nbytes),
                "ms_per_step": e2e_ms,
                "h2d_split": f"each rank copies 24n/{ws} bytes; NVLink all-gather assembles "
                             "the cloud (multigpu.gather_input)"},
        "gpu_launches": launches, "roofline": None, "cpu_baseline": None, "clocks": clk,
        "rank0_phases_ms": phases,
        "rank_memory_gb_estimate": {k: round(v / 1e9, 3) for k, v in
                                    MG.rank_memory_bytes(n, ws, max(2, plan.S // 10)).items()},
        "note": "roofline and cpu_baseline are on the N=1 line; rank0_phases_ms: one untimed "
                "call, presort / slab levels / cross levels (device events); "
                "rank_memory_gb_estimate: per-rank device bytes from the library's sizing "
                "functions (slab groups assumed <= S/10 kept points)",
    }
    print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
