#!/usr/bin/env python
"""Benchmark: residual samples/s (and Mrays/s) of the B200 residual path integral renderer.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

One step = one complete rr_render_residual of the workload (every enabled technique, both sides of the
two-way estimator) over this rank's sample shard, followed for N > 1 by the single NCCL
reduce of the residual image.  Inputs (scene + LBVH) are resident in HBM when the timed region
starts; the BVH (~350 MB for config 4) is larger than the 126 MB L2, so no flush is needed.  Rank 0 prints
ONE JSON line.  Under torchrun (N > 1) every rank renders its block-cyclic shard of sample indices.

--impl reference times the CPU oracle (oracle/, single-threaded fp64 C++) on the host cores on a bounded
sample of the same workload; it is the reference arm of the driver's comparison, not the target.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from rr_inputs import scenes as S  # noqa: E402


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=4)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=1)
    return p.parse_args()


def workload(cfg: int):
    return S.load_config(cfg)


def techniques_in(w) -> int:
    mask = w.args.technique_mask
    moved = any(not np.array_equal(e.old_xform, e.new_xform) for e in w.edits)
    if not moved:
        mask &= ~0x38
    return bin(mask).count("1")


def samples_per_render(w) -> int:
    c = w.scene.camera
    return techniques_in(w) * c.width * c.height * w.args.spp


# ---------------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region (B200_PROFILING.md)."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def rd():
            for line in self.proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])
        self.thread = threading.Thread(target=rd, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for n, v in zip(names, r[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------------- oracle
_ORACLE = None


def _oracle_worker(job):
    l, side, i0, i1 = job
    t = time.perf_counter()
    _, _, st = _ORACLE.residual(_ARGS, l, side, i0, i1)
    return time.perf_counter() - t, i1 - i0, st["closest_rays"] + st["shadow_rays"]


ORACLE_PER_TECH = 4096   # indices per (technique, side) per timed sample (2^12)
ORACLE_CHUNK = 256       # ... in chunks at seeded random positions over the whole index range
ORACLE_PER_TECH_1CORE = 512


def oracle_jobs(w, per_tech: int, seed: int = 0):
    """(technique, side, i0, i1) chunks of about per_tech indices per (technique, side), spread over the WHOLE
    index range (T7's pixel is i mod N_pix: every image row; the moved object at the image centre included)"""
    mask = _ORACLE.effective_mask(w.args.technique_mask)
    n_all = _ORACLE.sample_range(w.args)
    rng = np.random.default_rng(seed)
    jobs = []
    for l in range(1, 8):
        if (mask >> (l - 1)) & 1:
            for s in _ORACLE.sides(w.args):
                k = max(1, per_tech // ORACLE_CHUNK)
                starts = np.sort(rng.choice(max(1, n_all // ORACLE_CHUNK), size=k, replace=False)) * ORACLE_CHUNK
                jobs += [(l, s, int(a), int(min(a + ORACLE_CHUNK, n_all))) for a in starts]
    return jobs


class OracleTimer:
    """The oracle as it stands (single-threaded fp64 C++), on `cores` host processes.  The scene is loaded and
    the fork pool started and warmed BEFORE the timer; the timed region is the pool's map over the jobs only
    (counter-based RNG: disjoint index ranges are exact)."""

    def __init__(self, w, cores: int):
        global _ORACLE, _ARGS
        import multiprocessing as mp
        from oracle import binding as OB
        _ORACLE = OB.Oracle(w.scene, w.edits)
        _ARGS = w.args
        self.w, self.cores = w, cores
        self.pool = mp.get_context("fork").Pool(cores) if cores > 1 else None
        if self.pool:
            self.pool.map(_oracle_worker, [(7, 0, k, k + 1) for k in range(cores)])  # warm every worker

    def time(self, per_tech: int, seed: int = 0):
        jobs = oracle_jobs(self.w, per_tech, seed)
        t0 = time.perf_counter()
        res = self.pool.map(_oracle_worker, jobs, chunksize=1) if self.pool else [_oracle_worker(j) for j in jobs]
        wall = time.perf_counter() - t0
        return sum(r[1] for r in res), sum(r[2] for r in res), wall

    def close(self):
        if self.pool:
            self.pool.close()
            self.pool.join()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(w, steps: int = 1):
    """{1-core and all-core oracle samples/s on strided samples of the workload}"""
    cores = cpu_cores()
    one = OracleTimer(w, 1)
    n1, _, t1 = one.time(ORACLE_PER_TECH_1CORE, seed=1)
    allc = OracleTimer(w, cores)
    n, rays, wall = 0, 0, 0.0
    for k in range(steps):
        a, b, c = allc.time(ORACLE_PER_TECH, seed=100 + k)
        n, rays, wall = n + a, rays + b, wall + c
    allc.close()
    return {"value": n / wall, "unit": "samples/s", "cores": cores, "kind": "oracle",
            "sample": f"{ORACLE_PER_TECH} indices of every (technique, side) in chunks of {ORACLE_CHUNK} at seeded "
                      f"random positions over the whole index range of {w.name}, x{steps}",
            "mrays_per_s": rays / wall / 1e6, "one_core_samples_per_s": n1 / t1,
            "one_core_sample": f"{ORACLE_PER_TECH_1CORE} strided indices per (technique, side)",
            "cpu_model": cpu_model(), "cpu_seconds": wall * cores}


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = workload(a.config)
    cores = cpu_cores()
    per_tech = ORACLE_PER_TECH
    c = w.scene.camera
    timer = OracleTimer(w, cores)
    vals = []
    for k in range(a.warmup + a.steps):  # each step: a fresh strided sample of the workload
        n, rays, wall = timer.time(per_tech, seed=100 + k)
        if k >= a.warmup:
            vals.append((n, rays, wall))
    timer.close()
    n = sum(v[0] for v in vals)
    wall = sum(v[2] for v in vals)
    rays = sum(v[1] for v in vals)
    value = n / wall
    line = {
        "impl": "reference", "metric": "residual_samples_per_s", "value": value, "unit": "samples/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * wall / max(1, a.steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "scene": w.scene.name, "resolution": [c.width, c.height], "spp": w.args.spp,
                   "max_depth": w.args.max_depth,
                   "sample": f"{per_tech} strided indices of each (technique, side) per step (chunks of {ORACLE_CHUNK})"},
        "mrays_per_s": rays / wall / 1e6,
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "oracle",
                         "sample": f"{per_tech} indices of each (technique, side) in chunks of {ORACLE_CHUNK} at seeded "
                                   f"random positions over the whole index range, {a.steps} timed steps",
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------- ours
def run_ours(a):
    import torch
    import torch.distributed as dist
    from paper_2406_16302_b200 import Renderer, native  # noqa: F401
    from paper_2406_16302_b200.shard import reduce_image

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    w = workload(a.config)
    args = w.args
    c = w.scene.camera
    # CPU baseline (the oracle on the host cores) first, rank 0 at N = 1 only: before this process touches CUDA,
    # so the oracle's fork pool never forks a CUDA context
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(w)
    r = Renderer(local)
    t0 = time.time()
    r.upload(w.scene)
    r.set_edit(w.edits)
    torch.cuda.synchronize(dev)
    upload_s = time.time() - t0
    img = torch.empty((c.height, c.width, 4), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        r.render_residual(args, image=img, shard_index=rank, shard_count=world)
        reduce_image(img, dst=0)  # the one collective of the path (NCCL over NVLink), SURVEY 8(e)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize(dev)
    # ---- timed region (device events on the render stream, max over ranks)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats_acc = {"closest_rays": 0, "shadow_rays": 0, "nodes_visited": 0, "tris_tested": 0, "samples": 0}
    kern_ms = 0.0
    launches = 0
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    # per-step counters and per-launch kernel times of the last step (same work every step)
    st = r.get_stats()
    tm = r.last_timings(16)
    launch_ms = [x for x in tm[1:15] if x > 0]
    launches = len(launch_ms)
    sorted_launches = int(r.get_stats()["sched"][1])  # launches with the sample-ordering pre-pass (key kernel + sort)
    kern_ms = sum(launch_ms)
    for k in stats_acc:
        stats_acc[k] = st[k]
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    cnt = torch.tensor([float(stats_acc[k]) for k in ("closest_rays", "shadow_rays", "nodes_visited", "tris_tested",
                                                       "samples")], dtype=torch.float64, device=dev)
    kt = torch.tensor([kern_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
        dist.all_reduce(kt, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    closest, shadow, nodes, tris, samples = [float(x) for x in cnt.tolist()]
    total_samples = samples_per_render(w)
    assert abs(samples - total_samples) < 0.5, (samples, total_samples)
    value = total_samples * a.steps / (ms / 1e3)
    mrays = (closest + shadow) * a.steps / (ms / 1e3) / 1e6
    # ---- roofline of the dominant kernel: the (technique, both sides) launches with the largest time share.
    # Its algorithmic bytes = 64 B per BVH2 node fetched + 48 B per triangle tested, counted by
    # the kernels in an extra (untimed) render of exactly those launches: the full technique mask (same MIS and
    # pairing) with layer_mask = that technique.
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        peaks = json.load(open(peaks_path))
        hbm = float(peaks["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        hbm, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    mask = st["effective_mask"]
    sides = 2 if (args.flags & 1) else 1
    launch_tech = [l for l in range(1, 8) if (mask >> (l - 1)) & 1 for _ in range(sides)]
    per_tech_ms = {}
    for l, x in zip(launch_tech, tm[1:1 + len(launch_tech)]):
        per_tech_ms[l] = per_tech_ms.get(l, 0.0) + x
    dom = max(per_tech_ms, key=per_tech_ms.get)

    def counts(layer):  # untimed render with traversal counting (layer 0: every launch of the step)
        r.render_residual(dataclasses.replace(args, layer_mask=layer), image=img, shard_index=rank,
                          shard_count=world, count_traversal=True)
        q = r.get_stats()
        return q["nodes_visited"], q["tris_tested"]

    nodes, tris = counts(0)
    nd, td = counts(1 << (dom - 1))
    dom_bytes = 64.0 * nd + 48.0 * td                    # per render = both side launches
    dom_ms = per_tech_ms[dom]
    dom_launch_ms = dom_ms / sides
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else None
    kname = "k_residual_bidir" if dom in (3, 6) else "k_residual_single"
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": (achieved / hbm) if achieved else None, "traffic": None,
                "kernel": f"{kname} T{dom} (per launch: one side)", "peak_source": peak_src,
                "algorithmic_bytes_per_launch": dom_bytes / sides, "launch_ms": dom_launch_ms,
                "share_of_step": dom_ms / sum(per_tech_ms.values()),
                "all_launches": {"algorithmic_bytes_per_step": 64.0 * nodes + 48.0 * tris,
                                 "kernel_ms_per_step": float(kt.item()),
                                 "achieved_gbs": (64.0 * nodes + 48.0 * tris) / (float(kt.item()) / 1e3) / 1e9}}
    ncu = os.path.join(ROOT, "profiles", "ncu_t6_metrics.json")  # binding-resource counters
    if os.path.exists(ncu):
        try:
            roofline["ncu"] = json.load(open(ncu)).get(f"config{a.config}_T{dom}")
        except Exception:
            pass
    prof = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(prof):
        try:
            tr = json.load(open(prof)).get(f"config{a.config}_T{dom}")
            if tr:
                roofline["traffic"] = tr["dram_bytes_per_launch"]
                roofline["traffic_source"] = tr["source"]
        except Exception:
            pass
    # ---- end to end through the public API with host buffers (one render per step): each rank uploads its
    # per-step input (the edit), renders its shard into HOST memory (rr_render_residual_host), and for N > 1
    # the host images are summed on rank 0 (pinned host -> device, the NCCL reduce, device -> host).  Time =
    # max over ranks of the wall time of the loop.
    host = np.zeros((c.height, c.width, 4), np.float32)
    r.render_residual_host(args, out=host, shard_index=rank, shard_count=world)  # warm
    dev_img = torch.empty((c.height, c.width, 4), dtype=torch.float32, device=dev) if world > 1 else None
    pinned = torch.from_numpy(host).pin_memory() if world > 1 else None
    if world > 1:
        dist.barrier()
    t1 = time.perf_counter()
    for _ in range(a.e2e_steps):
        r.set_edit(w.edits)                                                         # host -> device input
        r.render_residual_host(args, out=host, shard_index=rank, shard_count=world)  # render + device -> host
        if world > 1:
            pinned.copy_(torch.from_numpy(host))
            dev_img.copy_(pinned, non_blocking=True)
            reduce_image(dev_img, dst=0)
            if rank == 0:
                pinned.copy_(dev_img)
    torch.cuda.synchronize(dev)
    el = torch.tensor([time.perf_counter() - t1], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    h2d = len(w.edits) * C_sizeof_edit() + C_sizeof_args() + (int(host.nbytes) if world > 1 else 0)
    d2h = int(host.nbytes) * (2 if world > 1 and rank == 0 else 1)
    e2e = {"value": total_samples * a.e2e_steps / float(el.item()), "unit": "samples/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
    if rank == 0:
        line = {
            "metric": "residual_samples_per_s", "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": w.name, "scene": w.scene.name, "triangles": w.scene.n_triangles,
                       "resolution": [c.width, c.height], "spp": args.spp, "max_depth": args.max_depth,
                       "techniques": techniques_in(w), "flags": "two_way+reconnect+reject_multi",
                       "samples_per_step": total_samples, "parallelism": f"sample-shard x{world} + NCCL reduce",
                       "l2": "inputs larger than L2 (BVH ~350 MB vs 126 MB L2)"},
            "mrays_per_s": mrays,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            # residual kernels + our sample-key kernels; each key kernel is followed by one CUB radix sort
            # (library kernels, not counted here); ordering pre-passes take ordering_ms_per_step of the step
            "gpu_launches": (launches + sorted_launches) * a.steps,
            "cub_radix_sorts_per_step": sorted_launches,
            "ordering_ms_per_step": float(tm[15]),
            "clocks": clk,
            "upload_s": upload_s,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def C_sizeof_edit() -> int:
    import ctypes
    from paper_2406_16302_b200 import native
    return ctypes.sizeof(native.rr_edit)


def C_sizeof_args() -> int:
    import ctypes
    from paper_2406_16302_b200 import native
    return ctypes.sizeof(native.rr_render_args)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
