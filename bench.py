#!/usr/bin/env python
"""Benchmark: docked ligands/s of the B200 pose-search path (BASELINE config 1).

One step = one pass of the hot path over one batch: every ligand of the
rank's shard goes through the rigid sweep, top-K selection, K restart
chains of fragment optimisation, and the final ordering (E1-E8).

* ``value``: device-resident throughput -- descriptors already in HBM, CUDA
  events around each step's kernels (and, for N > 1, the NCCL top-K gather),
  L2 flushed between steps.
* ``e2e``: the same metric through the public C-ABI call (gd_dock_batch)
  with host buffers: host preprocessing, pinned H2D, kernels, D2H.
* ``--impl reference``: the reference's own CPU path (oracle/_ref: the
  reference headers compiled from /root/reference, PocketIndex, all host
  threads) on a bounded sample of the same workload.
* ``--workload profiles``: the analysis row -- rotation
  profiles (analysis.hpp:37-56, 360 integer angles per fragment) of every
  fragment of the config's ligands from their given poses; metric
  fragments/s, same keys (roofline of the profile kernel, e2e through
  gd_upload + gd_rotation_profiles, the reference's rotation_profile on the
  host cores as cpu_baseline / --impl reference).

Multi-GPU (torchrun): ligands are sharded by id (weak scaling: every rank
docks its own seeded 10,000); each step all-gathers every rank's per-ligand
top-K table over NCCL from device memory.
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "docked ligands/sec and poses scored/sec at 1/2/4/8 B200 vs host-core CPU ref"
# Algorithmic fp64 FLOPs per unit of counted work.
FLOPS = {"pairs": 9, "rotated": 36, "bump_pairs": 11, "queries": 0, "sum_terms": 2,
         "evaluations": 2, "xform": 18}
CPU_SAMPLE = 256  # ligands of the shard timed on the host cores


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--ligands", type=int, default=0, help="override ligands per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--workload", default="dock", choices=["dock", "profiles"])
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class Clocks:
    """nvidia-smi sampler for the timed region (median SM clock, reasons)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.rows = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 "100", "-i", str(device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower() in ("active", "1")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


L2_NOTE = ("flushed between steps, untimed: a 256 MiB write, then a 256 MiB read sweep so the "
           "flush's dirty lines are written back before the timed region, not during it")


def flush_l2(buf) -> None:
    """Evict the 126 MB L2 (256 MiB write), then read the buffer back so no
    dirty flush line is written back inside the next timed kernel."""
    buf.zero_()
    buf.sum()


def flops_of(work: dict) -> float:
    return float(sum(FLOPS[k] * v for k, v in work.items()))


CPU_BRUTE_SAMPLE = 24  # ligands of the brute-force (no PocketIndex) reference timing


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference(batch, pocket, knobs, n: int, brute: bool = False):
    """The reference CPU path on the first n ligands: (ligands/s, info).
    brute: the reference's default brute-force overlap scan instead of its
    PocketIndex (the CLI's --spatial-index path, tools/geodock.cpp:387)."""
    from oracle import oracle_py as O
    sub = batch.subset(range(min(n, batch.n_ligands)))
    threads = O.threads()
    kind = "reference" if O.have_ref() else "port"
    impl = "ref" if kind == "reference" else "oracle"
    t0 = time.perf_counter()
    res = O.dock_batch(sub, pocket, knobs, nthreads=threads, keep_poses=False, impl=impl,
                       use_index=not brute)
    dt = time.perf_counter() - t0
    return sub.n_ligands / dt, {
        "kind": kind, "cores": threads, "cpu_model": cpu_model(), "logical_cpus": os.cpu_count(),
        "sample": (f"first {sub.n_ligands} ligands of the workload, "
                   + (("reference headers (oracle/_ref) with "
                       + ("brute-force scan" if brute else "PocketIndex"))
                      if kind == "reference" else "C oracle")
                   + f", {threads} threads"),
        "poses_scored_per_s": float(res.poses_scored.sum()) / dt, "seconds": dt}


def cpu_baseline_of(batch, pocket, knobs) -> dict:
    """cpu_baseline: PocketIndex on CPU_SAMPLE ligands (the value) and the
    brute-force scan on CPU_BRUTE_SAMPLE beside it."""
    v, inf = cpu_reference(batch, pocket, knobs, CPU_SAMPLE)
    vb, infb = cpu_reference(batch, pocket, knobs, CPU_BRUTE_SAMPLE, brute=True)
    return {"value": v, "unit": "ligands/s", "cores": inf["cores"], "kind": inf["kind"],
            "sample": inf["sample"], "cpu_model": inf["cpu_model"], "logical_cpus": inf["logical_cpus"],
            "brute_force": {"value": vb, "unit": "ligands/s", "sample": infb["sample"]}}


def reference_inputs() -> None:
    """Inputs of the reference arms come from the generator built on its own
    (oracle/libgd_synth.so, same csrc/synth.cpp): they never load the
    product library."""
    from oracle import oracle_py as O
    if not (O.HERE / "libgd_synth.so").exists():
        O.build(ref=True)
    from paper_1901_06363_b200 import native
    native.set_synth_library(O.HERE / "libgd_synth.so")


def assert_no_product_library() -> None:
    maps = Path("/proc/self/maps").read_text()
    assert "libgeodock_b200" not in maps, "a reference arm loaded the product library"


def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    reference_inputs()
    from paper_1901_06363_b200 import workloads as W
    w = W.config(a.config)
    pocket = w.pocket()
    n = a.ligands or CPU_SAMPLE
    batch = w.ligands(range(n), pocket.mean(axis=0))
    for _ in range(a.warmup):
        cpu_reference(batch, pocket, w.knobs, n)
    info = None
    t0 = time.perf_counter()
    for _ in range(a.steps):
        _, info = cpu_reference(batch, pocket, w.knobs, n)
    wall = time.perf_counter() - t0
    value = n * a.steps / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "ligands/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * wall / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "ligands_per_step": n},
        "cpu_baseline": {"value": value, "unit": "ligands/s", "cores": info["cores"],
                         "kind": info["kind"], "sample": info["sample"],
                         "cpu_model": info["cpu_model"], "logical_cpus": info["logical_cpus"]},
        "e2e": {"value": value, "unit": "ligands/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    assert_no_product_library()
    print(json.dumps(line), flush=True)


def run_ours(a):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1901_06363_b200 import Docker, Knobs, workloads as W
    from paper_1901_06363_b200.native import DockResult, GD_FLAG_COUNT_WORK
    from paper_1901_06363_b200.sharding import DeviceGather, shard_ids

    w = W.config(a.config)
    pocket = w.pocket()
    n_per = a.ligands or w.n_ligands
    batch = w.ligands(shard_ids(rank, world, n_per, "weak"), pocket.mean(axis=0))
    knobs = w.knobs
    K = knobs.slots

    # A dedicated stream for everything in the timed loop (the flush, the
    # events, the library's kernels): torch's default stream is handle 0,
    # which gd_set_stream reads as "the context's own stream", so events on
    # it would not order the kernels.
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    d = Docker(local)
    d.set_stream(stream.cuda_stream)
    d.set_pocket(pocket)
    info = d.pocket_info()
    d.upload(batch)

    # One counted, untimed step: exact executed work per launch.
    d.dock_resident(Knobs(**{**knobs.__dict__, "flags": GD_FLAG_COUNT_WORK}))
    work = d.work_counters()
    fp64_peak = d.fp64_peak_tflops()
    l2_peak = d.l2_gather_peak_gbs()
    l2_at_occ = d.l2_gather_rate_gbs(24)  # the flex kernel's residency, one gather in flight per lane

    d.dock_resident(knobs)
    gather = DeviceGather(d.device_results(), world) if world > 1 else None
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def step():
        d.dock_resident(knobs, top_pose=True)  # the same work as the e2e call (top-1 poses kept)
        if gather is not None:
            gather()  # NCCL all-gather of every rank's top-K table

    for _ in range(a.warmup):
        step()
    rigid_ms, flex_ms, step_ms = [], [], []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    for _ in range(a.steps):
        flush_l2(flush)  # untimed: evicts the 126 MB L2 between steps
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        t = d.timing()
        rigid_ms.append(t["rigid_ms"])
        flex_ms.append(t["flex_ms"])
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    total_ms = float(sum(step_ms))
    if dist:
        tt = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / a.steps
    value = world * batch.n_ligands / (ms_per_step / 1e3)

    res = d.download(DockResult.empty(batch.n_ligands, K, int(batch.atom_offsets[-1]), False))
    poses_per_step = float(res.poses_scored.sum())
    # executed point pairs vs the brute-force scan's n*P per scored pose.
    brute_pairs = float((res.poses_scored * batch.sizes).sum()) * len(pocket)
    exec_pairs = float(work["rigid"]["pairs"] + work["flex"]["pairs"])
    if dist:
        ps = torch.tensor([poses_per_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(ps)
        poses_per_step = float(ps.item())
    poses_per_s = poses_per_step / (ms_per_step / 1e3)

    # e2e: host buffers through gd_dock_batch (prep + pinned H2D + kernels + D2H).
    e2e = None
    if not a.no_e2e:
        e2e_steps = max(1, min(a.steps, 5))
        # warm; host result arrays reused, as a caller would; every field of
        # the top-K table plus each ligand's top-1 pose comes back
        host_out = d.dock(batch, knobs, top_pose=True)
        tms = []
        for _ in range(e2e_steps):
            flush_l2(flush)
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            d.dock(batch, knobs, out=host_out, top_pose=True)
            tms.append(time.perf_counter() - t0)
        tt = float(np.mean(tms))
        if dist:
            x = torch.tensor([tt], device="cuda", dtype=torch.float64)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            tt = float(x.item())
        tim = d.timing()
        e2e = {"value": world * batch.n_ligands / tt, "unit": "ligands/s",
               "h2d_bytes_per_step": int(tim["h2d_bytes"]),
               "d2h_bytes_per_step": int(tim["d2h_bytes"]), "ms_per_step": 1e3 * tt,
               "steps": e2e_steps, "timer": "host wall clock around gd_dock_batch",
               "returns": "top-K table (orientation, seed rank, rigid/final score, evaluations, "
                          "feasibility checks), k_eff, poses scored, status, top-1 pose"}

    if rank == 0:
        r_ms, f_ms = float(np.mean(rigid_ms)), float(np.mean(flex_ms))
        dom = "flex_chain_kernel" if f_ms >= r_ms else "rigid_topk_kernel"
        dom_work = work["flex" if dom == "flex_chain_kernel" else "rigid"]
        dom_ms = max(r_ms, f_ms)
        achieved = flops_of(dom_work) / (dom_ms / 1e3) / 1e12
        # DRAM traffic per launch from the committed ncu --set full capture of
        # this exact workload (ncu cannot run inside the bench itself).
        traffic, traffic_src = None, None
        tj = ROOT / "profiles" / "ncu_traffic.json"
        if tj.exists():
            tr = json.loads(tj.read_text())
            if tr.get("config") == a.config and tr.get("ligands_per_gpu") == batch.n_ligands:
                traffic = tr["dram_bytes_per_launch"].get(dom)
                traffic_src = tr["source"]
        line = {
            "metric": METRIC, "value": value, "unit": "ligands/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE generators, DESIGN.md §5)",
            "config": {"workload": w.name, "ligands_per_gpu": batch.n_ligands,
                       "pocket_points": len(pocket), "rigid_step": knobs.rigid_step,
                       "fragment_step": knobs.high_precision_step,
                       "restarts": knobs.repetitions, "top_k": knobs.top_k,
                       "parallelism": f"ligand-sharded x{world}" + (", NCCL top-K all-gather per step"
                                                                    if world > 1 else ""),
                       "l2": L2_NOTE,
                       "voxel_index": {k: (v.tolist() if hasattr(v, "tolist") else v)
                                       for k, v in info.items()}},
            "poses_scored_per_s": poses_per_s,
            "pairs": {"executed_per_s": world * exec_pairs / (ms_per_step / 1e3),
                      "brute_equivalent_per_s": world * brute_pairs / (ms_per_step / 1e3),
                      "index_pruning_ratio": brute_pairs / max(exec_pairs, 1.0),
                      "note": "a work ratio, not a throughput: brute-force equivalent = n_atoms x "
                              "pocket points per scored pose (the reference's distance_sq calls "
                              "without PocketIndex) over the point pairs the exact voxel index "
                              "actually evaluates"},
            "kernel_ms": {"rigid_topk_kernel": r_ms, "flex_chain_kernel+finalize": f_ms},
            "gpu_launches": 3 * a.steps,
            "roofline": {"kernel": dom, "bound": "fp64", "achieved": achieved,
                         "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                         "traffic": traffic, "traffic_unit": "bytes per launch (DRAM read+write)",
                         "traffic_source": traffic_src,
                         "peak_source": "measured fp64 DADD/DMUL probe (gd_fp64_peak) on this GPU",
                         "work_per_launch": dom_work},
            # North star: the fraction of the L2-gather roofline.  Every
            # candidate point costs one 32-byte index gather (its voxel record
            # or list entry); peak = the same access pattern measured alone.
            "roofline_l2_gather": {"kernel": dom, "bound": "l2",
                                   "achieved": 32.0 * dom_work["pairs"] / (dom_ms / 1e3) / 1e9,
                                   "peak": l2_peak, "unit": "GB/s",
                                   "frac": 32.0 * dom_work["pairs"] / (dom_ms / 1e3) / 1e9 / l2_peak,
                                   "peak_source": "measured random 32 B L1-bypassing gathers over "
                                                  "an L2-resident 48 MB buffer (gd_l2_gather_peak)",
                                   "latency_bound_at_residency": {
                                       "gbs": l2_at_occ,
                                       "frac": 32.0 * dom_work["pairs"] / (dom_ms / 1e3) / 1e9 / l2_at_occ,
                                       "what": "the same gathers with one dependent load in flight per "
                                               "lane at the flex kernel's 24 warps per SM "
                                               "(gd_l2_gather_rate): the ceiling for lanes that each "
                                               "wait on their own lookup"}},
            "clocks": clk,
        }
        if e2e:
            line["e2e"] = e2e
        if world == 1 and not a.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_of(batch, pocket, knobs)
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


PROFILE_METRIC = "fragment rotation profiles/s (360 integer angles each, analysis.hpp rotation_profile)"
PROFILE_LIGANDS = 2000  # ligands per step (about 9,000 fragments on config 1)
PROFILE_CPU_SAMPLE = 256


def cpu_profiles(batch, pocket, n: int):
    """The reference's rotation_profile on the first n ligands: (fragments/s, info)."""
    from oracle import oracle_py as O
    sub = batch.subset(range(min(n, batch.n_ligands)))
    threads = O.threads()
    kind = "reference" if O.have_ref() else "port"
    t0 = time.perf_counter()
    out = O.rotation_profiles(sub, pocket, "ref" if kind == "reference" else "oracle",
                              nthreads=threads)
    dt = time.perf_counter() - t0
    return len(out[0]) / dt, {
        "kind": kind, "cores": threads if kind == "reference" else 1,
        "sample": (f"first {sub.n_ligands} ligands ({len(out[0])} fragments) of the workload, "
                   + ("reference rotation_profile (oracle/_ref) with PocketIndex"
                      if kind == "reference" else "C oracle, brute force")),
        "seconds": dt}


def profile_batch_of(a):
    from paper_1901_06363_b200 import workloads as W
    w = W.config(a.config)
    pocket = w.pocket()
    n = a.ligands or PROFILE_LIGANDS
    return w, pocket, w.ligands(range(n), pocket.mean(axis=0))


def run_profiles_reference(a):
    rank, _, _ = dist_env()
    if rank != 0:
        return
    reference_inputs()
    w, pocket, batch = profile_batch_of(a)
    for _ in range(a.warmup):
        cpu_profiles(batch, pocket, PROFILE_CPU_SAMPLE)
    t0 = time.perf_counter()
    frags = 0
    info = None
    for _ in range(a.steps):
        v, info = cpu_profiles(batch, pocket, PROFILE_CPU_SAMPLE)
        frags += v * info["seconds"]
    wall = time.perf_counter() - t0
    value = frags / wall
    print(json.dumps({
        "impl": "reference", "metric": PROFILE_METRIC, "value": value, "unit": "fragments/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * wall / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"profiles of {w.name}", "ligands_per_step": PROFILE_CPU_SAMPLE},
        "cpu_baseline": {"value": value, "unit": "fragments/s", "cores": info["cores"],
                         "kind": info["kind"], "sample": info["sample"], "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "fragments/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)
    assert_no_product_library()


def run_profiles(a):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    from paper_1901_06363_b200 import Docker
    from paper_1901_06363_b200.native import GD_FLAG_COUNT_WORK
    w, pocket, batch = profile_batch_of(a)
    stream = torch.cuda.Stream()  # see run_ours
    torch.cuda.set_stream(stream)
    d = Docker(local)
    d.set_stream(stream.cuda_stream)
    d.set_pocket(pocket)
    d.upload(batch)
    prof = d.rotation_profiles(flags=GD_FLAG_COUNT_WORK)  # counted, untimed
    work = d.work_counters()["flex"]
    F = len(prof.scores)
    fp64_peak = d.fp64_peak_tflops()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    from paper_1901_06363_b200.native import ProfileBuffers
    out = ProfileBuffers.for_batch(batch)  # host outputs reused across steps, as a caller would
    for _ in range(a.warmup):
        d.rotation_profiles(out=out)
    kern_ms, call_ms = [], []
    torch.cuda.synchronize()
    clocks = Clocks(local)
    for _ in range(a.steps):
        flush_l2(flush)
        torch.cuda.synchronize()
        d.rotation_profiles(out=out)
        t = d.timing()
        kern_ms.append(t["flex_ms"])
        call_ms.append(t["total_ms"])
    clk = clocks.stop()
    ms = float(np.mean(kern_ms))
    value = F / (ms / 1e3)
    e2e = None
    if not a.no_e2e:
        tms = []
        for _ in range(max(1, min(a.steps, 5))):
            flush_l2(flush)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            d.rotation_profiles(batch, out=out)  # host prep + H2D + kernel + D2H of 360 x 9 B per fragment
            tms.append(time.perf_counter() - t0)
        tt = float(np.mean(tms))
        t = d.timing()
        e2e = {"value": F / tt, "unit": "fragments/s",
               "h2d_bytes_per_step": int(batch.xyz.nbytes + batch.radii.nbytes + t["h2d_bytes"]),
               "d2h_bytes_per_step": int(t["d2h_bytes"]), "ms_per_step": 1e3 * tt,
               "timer": "host wall clock around gd_upload + gd_rotation_profiles"}
    achieved = flops_of(work) / (ms / 1e3) / 1e12
    line = {
        "metric": PROFILE_METRIC, "value": value, "unit": "fragments/s", "n_gpus": 1,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generators, DESIGN.md §5)",
        "config": {"workload": f"profiles of {w.name} (given poses)",
                   "ligands": batch.n_ligands, "fragments": F, "angles_per_fragment": 360,
                   "pocket_points": len(pocket),
                   "l2": L2_NOTE},
        "kernel_ms": {"profile_kernel": ms}, "call_ms": float(np.mean(call_ms)),
        "gpu_launches": a.steps,
        "roofline": {"kernel": "profile_kernel", "bound": "fp64", "achieved": achieved,
                     "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                     "traffic": None, "peak_source": "measured fp64 DADD/DMUL probe (gd_fp64_peak)",
                     "work_per_launch": work},
        "clocks": clk,
    }
    if e2e:
        line["e2e"] = e2e
    if not a.no_cpu_baseline:
        v, inf = cpu_profiles(batch, pocket, PROFILE_CPU_SAMPLE)
        line["cpu_baseline"] = {"value": v, "unit": "fragments/s", "cores": inf["cores"],
                                "kind": inf["kind"], "sample": inf["sample"]}
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = args_()
    if a.workload == "profiles":
        run_profiles_reference(a) if a.impl == "reference" else run_profiles(a)
    elif a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
