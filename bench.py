#!/usr/bin/env python
"""Benchmark of the B200 correction loop (BASELINE.json metric: Mvertices/s of
end-to-end correction to convergence; per-kernel HBM GB/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

A "step" is one full derive_edits (validation → C/R loops to convergence →
postconditions → EditSet compaction) over one synthetic field.

* value  — device-resident: f and f̂ already in HBM, EditSet left in HBM;
           CUDA events on the caller stream around every step (L2 flushed
           between steps by a 512 MB write outside the events); max over ranks.
* e2e    — the public host API (derive_edits_into) from pinned host buffers:
           H2D of f and f̂ plus D2H of the EditSet inside the timed region.
* roofline — the graded kernel (the streaming class with the most device
           time, picked from one fully profiled warm-up step), from per-launch
           CUDA events on the engine's stream during the timed steps (only that
           class is event-timed there), achieved = algorithmic bytes per launch
           / mean launch time; per_class and kernel_profile_ms_per_step come
           from the profiled warm-up step.
* cpu_baseline — the UNMODIFIED reference (oracle/_ref/libmssz_ref.so,
           OpenMP, all host cores) on a bounded sample of the same workload.

N > 1 (torchrun), 3D configs: the field is z-slab sharded, one slab per rank
(SURVEY §8(e), strong scaling: the total field is fixed).  Rank 0 generates the
field and sends every rank its window (owned planes + 2 halo planes per side)
over NCCL before timing; each step is one sharded derive_edits through
mssz_cu_derive_edits_slab_device (value) / mssz_cu_derive_edits_slab (e2e).
2D configs at N > 1 run one replica per rank (weak scaling).
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mvertices/s end-to-end correction (to convergence)"
UNIT = "Mvertices/s"

# Algorithmic bytes of the timed steps per kernel class, from the
# step's own counters where a launch covers less than the whole field.  Classes
# without an entry (persistent subloop, gathers over lists) are latency-bound
# and not roofline-graded.
# Freudenthal rings (grid.cpp:8-16): |{t} ∪ N(t)| and |2-ring of t| (2D, 3D)
RING1 = {2: 7, 3: 15}
RING2 = {2: 19, 3: 65}


def alg_bytes(cls: str, es: int, n: int, st, launches: int, ndims: int = 3) -> float:
    tile = 8192
    r1, r2 = RING1[ndims], RING2[ndims]
    return {
        # persistent C loop (run_subloop, edit_engine.cpp:246-278), per worklist
        # item: list entry 4 + its code 1 + claim stamp 4 + next-list entry 4;
        # per applied edit: the lowered value written, the values of the 2-ring
        # of t (the inputs of every code the edit can change, mss.cpp:17-29) and
        # the 1-ring's codes (g code written, f code read for the kind test)
        "subloop": 13 * st.subloop_items + (es + r2 * es + 2 * r1) * st.subloop_edits,
        "validate": 2 * es * n * launches,               # read f and fhat
        "directions": (es + 1) * n * launches,           # read values, write one code byte
        "detect_kind": 2 * n * launches,                 # full sweeps: fdir + gdir
        "label_init": 9 * tile * st.label_tiles,         # code byte in, two u32 labels out per tile vertex
        "label_finish": 16 * n * launches,               # two labels read + gathered (f labels once)
        # both codes of every listed tile vertex; per divergent (vertex, family):
        # provisional label, its final (one gather) and the f label
        "rfix": 2 * tile * st.rfix_tiles + 12 * st.rfix_divergent,
        "compact": 2 * n * launches,                     # flag sweep (count + write passes)
    }.get(cls, 0.0)


# bounded CPU samples (about 5-20 s of reference work on 16 host cores)
CPU_SAMPLE = {
    "C1": (512, 512), "C2": (177, 95, 48), "C2-trig": (177, 95, 48),
    "C3": (96, 96, 96), "C4": (128, 128, 64), "C5": (720, 480),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--dims", default=None, help="override dims, e.g. 256x256x256")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--cpu-dims", default=None)
    ap.add_argument("--shard", action="store_true",
                    help="z-slab sharded path even at N=1 (one-rank NCCL communicator)")
    return ap.parse_args()


def dims_arg(s):
    return tuple(int(x) for x in s.lower().split("x")) if s else None


class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, use_cuda=True):
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            backend = "nccl" if use_cuda else "gloo"
            if use_cuda:
                import torch
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t)
        return float(t.item())

    def done(self):
        if self.pg:
            self.pg.destroy_process_group()


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.fp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.fp, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.fp.flush()
        self.fp.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.fp.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        os.unlink(self.fp.name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fp:
            d = json.load(fp)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_reference_run(cfg, dims, dtype, threads, steps=1, want_inputs=False):
    """The unmodified reference derive_edits on the host (oracle/_ref): returns
    (times, stats) or, with want_inputs, (times, stats, (f, fhat, xi), result)."""
    import oracle as O
    if not O.have_ref():
        raise RuntimeError("oracle/_ref/libmssz_ref.so missing (build() it in the build container)")
    R = O.ref()
    # inputs through the reference's own generator and codec
    if cfg.kind == "multi-scale":
        gm = R.generate("gaussian-mixture", list(dims), cfg.seed, np.float64)
        rs = R.generate("random-smooth", list(dims), cfg.seed + 1, np.float64)
        f = (gm + cfg.a * rs).astype(dtype)
    else:
        f = R.generate(cfg.kind, list(dims), cfg.seed, dtype)
    xi = R.resolve_rel(list(dims), f, cfg.rel)
    fh = R.compress_base(list(dims), f, xi)
    times, res = [], None
    for _ in range(steps):
        t = time.perf_counter()
        res = R.derive_edits(list(dims), f, fh, xi, subloop_cap=cfg.subloop_cap, threads=threads)
        times.append(time.perf_counter() - t)
    if want_inputs:
        return times, res.stats, (f, fh, xi), res
    return times, res.stats


STAT_KEYS = ("outer_iterations", "c_passes", "sub_iterations", "r_iterations",
             "effective_edits", "touched")


def same_input_comparison(P, cfg, sdims, inputs, ref_res, ref_s, device=0):
    """The B200 engine on exactly the reference arm's input (its own generator
    and base codec), through the public host API: EditStats side by side
    (edit_engine.hpp:54-68) and the same-input speed ratio."""
    f, fh, xi = inputs
    topo = P.build_topology(list(sdims))
    opts = P.DeriveOptions(subloop_cap=cfg.subloop_cap, device=device)
    P.derive_edits(topo, f, fh, xi, opts)  # warm (workspace sized)
    walls, st, e = [], None, None
    for _ in range(3):
        st = P.EditStats()
        t = time.perf_counter()
        e = P.derive_edits(topo, f, fh, xi, opts, st)
        walls.append(time.perf_counter() - t)
    gpu_s = min(walls)
    rt = ref_res.stats["touched"]
    gpu = {k: getattr(st, k) for k in STAT_KEYS}
    ref = {k: ref_res.stats[k] for k in STAT_KEYS}
    common = int(np.intersect1d(e.indices, ref_res.indices, assume_unique=True).size)
    return {
        "input": "identical arrays: the reference's generate_synthetic + compress_base outputs",
        "dims": list(sdims), "vertices": int(np.prod(sdims)),
        "gpu_edit_stats": gpu, "reference_edit_stats": ref,
        "touched_diff": int(st.touched) - int(rt), "touched_tolerance": max(4, int(1e-4 * rt)),
        "edit_sets_identical": bool(np.array_equal(e.indices, ref_res.indices)
                                   and e.values.tobytes() == ref_res.values.tobytes()),
        "edit_index_overlap": {"gpu": int(e.indices.size), "reference": int(ref_res.indices.size),
                               "common": common},
        "gpu_e2e_s": gpu_s, "reference_s": ref_s,
        "same_input_speedup_e2e": ref_s / gpu_s,
        "gpu_api": "derive_edits (mssz_cu_derive_edits, host buffers in and out)",
    }


def run_reference_arm(args, cfg, dist):
    if dist.rank != 0:
        return
    dims = dims_arg(args.cpu_dims) or CPU_SAMPLE.get(cfg.name, cfg.dims)
    dtype = np.float32 if args.dtype == "f32" else np.float64
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_WAIT_POLICY", "active")
    times, st = cpu_reference_run(cfg, dims, dtype, threads, steps=args.warmup + args.steps)
    timed = times[args.warmup:]
    n = int(np.prod(dims))
    mean = statistics.mean(timed)
    value = n / mean / 1e6
    sample = f"{cfg.name} kind={cfg.kind} at {'x'.join(map(str, dims))} ({n} vertices), rel {cfg.rel}"
    same = list(dims) == list(cfg.dims)
    workload = cfg.note if same else (
        f"bounded CPU sample of {cfg.name} ({cfg.note}): the same generator at "
        f"{'x'.join(map(str, dims))}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": mean * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": workload, "config_id": cfg.name, "config_dims": list(cfg.dims),
                   "sample_dims": list(dims), "same_config": same, "rel_eb": cfg.rel,
                   "subloop_cap": cfg.subloop_cap, "parallelism": f"openmp x{threads}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "edit_stats": st,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    from paper_2406_09423_b200 import inputs as I
    cfg = I.CONFIGS[args.config]
    dist = Dist()
    if args.impl == "reference":
        run_reference_arm(args, cfg, dist)
        return

    import torch
    import paper_2406_09423_b200 as P

    dist.init()
    torch.cuda.set_device(dist.local)
    dtype = np.float32 if args.dtype == "f32" else np.float64
    tdtype = torch.float32 if args.dtype == "f32" else torch.float64
    es = 4 if args.dtype == "f32" else 8
    dims = dims_arg(args.dims) or cfg.dims
    topo = P.build_topology(dims)
    n = topo.vertex_count

    t_gen = time.perf_counter()
    sharded = (dist.world > 1 or args.shard) and len(dims) == 3
    if sharded and dist.rank != 0:
        f = fh = xi = None  # sharded: rank 0 generates and sends the windows
    else:
        f, fh, xi = I.make_inputs(cfg, dims, dtype)
    t_gen = time.perf_counter() - t_gen

    dev = torch.device("cuda", dist.local)
    comm = None
    if sharded:
        # rank 0 holds the whole field; every rank receives its window over NCCL
        XY = dims[0] * dims[1]
        z0, z1, wz0, wz1 = P.slab_range(dims[2], dist.world, dist.rank)
        meta = [xi, P.SlabComm.unique_id() if dist.rank == 0 else None]
        if dist.pg:
            dist.pg.broadcast_object_list(meta, src=0)
        xi = meta[0]
        if dist.rank == 0:
            full = [torch.from_numpy(a).to(dev) for a in (f, fh)]
            for r in range(1, dist.world):
                _, _, a, b = P.slab_range(dims[2], dist.world, r)
                for t in full:
                    dist.pg.send(t[a * XY:b * XY].contiguous(), dst=r)
            df, dfh = (t[wz0 * XY:wz1 * XY].clone() for t in full)
            del full
        else:
            df = torch.empty((wz1 - wz0) * XY, dtype=tdtype, device=dev)
            dfh = torch.empty_like(df)
            for t in (df, dfh):
                dist.pg.recv(t, src=0)
        torch.cuda.synchronize()
        f = fh = None  # host copies of the window are made for the e2e leg below
        comm = P.SlabComm(meta[1], dist.world, dist.rank, dist.local)
        cap = (z1 - z0) * XY
        n_local = df.numel()
    else:
        df = torch.from_numpy(f).to(dev)
        dfh = torch.from_numpy(fh).to(dev)
        cap = n
        n_local = n
    d_idx = torch.empty(cap, dtype=torch.int64, device=dev)
    d_val = torch.empty(cap, dtype=tdtype, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    opts = P.DeriveOptions(subloop_cap=cfg.subloop_cap, device=dist.local)

    def step(profile=False):
        opts.profile = profile
        if comm is not None:
            c, _, s = comm.derive_edits_device(dims, df.data_ptr(), dfh.data_ptr(), xi,
                                               d_idx.data_ptr(), d_val.data_ptr(), cap, dtype,
                                               opts, stream.cuda_stream)
            return c, s
        return P.derive_edits_device(topo, df.data_ptr(), dfh.data_ptr(), xi, d_idx.data_ptr(),
                                     d_val.data_ptr(), cap, dtype, opts, stream.cuda_stream)

    # The last warm-up step times every kernel class (CUDA events around each
    # launch): it gives the per-class breakdown and picks the graded kernel.  The
    # timed steps then time only that class, so ~10k event records per step do
    # not inflate the headline; its roofline comes from the timed region.
    prof_stats = None
    for w in range(max(args.warmup, 0 if args.no_profile else 1)):
        last = w == max(args.warmup, 1) - 1
        count, st = step(profile=last and not args.no_profile)
        if last and not args.no_profile:
            prof_stats = st
    torch.cuda.synchronize()
    top = None
    if prof_stats is not None:
        kp = prof_stats.kernel_profile()
        cand = {k: v["ms"] for k, v in kp.items()
                if v["launches"] and alg_bytes(k, es, n_local, prof_stats, v["launches"], len(dims))}
        top = max(cand, key=cand.get) if cand else None
    timed_profile = P.profile_mask(top) if top else False

    dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(dist.local)
    step_ms, stats = [], []
    for _ in range(args.steps):
        flush.fill_(1.0)  # evict L2 between steps (outside the events)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        count, st = step(profile=timed_profile)
        b.record(stream)
        b.synchronize()
        step_ms.append(a.elapsed_time(b))
        stats.append(st)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    ms = dist.max(statistics.mean(step_ms))
    total_vertices = float(n) if sharded else dist.sum(float(n))
    value = total_vertices / (ms * 1e-3) / 1e6

    # ---- roofline of the dominant kernel class (live, from the timed steps)
    peak, peak_src = load_peaks()
    roofline = None
    prof = {}
    if prof_stats is not None:
        # per-class breakdown: the fully profiled warm-up step
        pk = prof_stats.kernel_profile()
        prof = {k: {"launches": v["launches"], "ms": v["ms"]} for k, v in pk.items() if v["launches"]}
    if prof_stats is not None and top is not None:
        total_ms = sum(v["ms"] for v in prof.values())
        graded = {}
        for k, v in prof.items():
            tot = alg_bytes(k, es, n_local, prof_stats, v["launches"], len(dims))
            if tot:
                graded[k] = {"launches": v["launches"], "ms": v["ms"], "bytes": tot,
                             "achieved_GBps": tot / (v["ms"] * 1e-3) / 1e9}
        # the graded kernel: achieved from its launches inside the timed steps
        t_launch = sum(s.kernel_profile()[top]["launches"] for s in stats)
        t_ms = sum(s.kernel_profile()[top]["ms"] for s in stats)
        t_bytes = sum(alg_bytes(top, es, n_local, s, s.kernel_profile()[top]["launches"], len(dims)) for s in stats)
        per_launch_ms = t_ms / t_launch
        bytes_per_launch = t_bytes / t_launch
        achieved = t_bytes / (t_ms * 1e-3) / 1e9
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic_c4.json")
        traffic = None  # measured DRAM bytes per launch of this kernel (committed ncu capture, same config)
        if cfg.name == "C4" and dims == cfg.dims and os.path.exists(tpath):
            with open(tpath) as fp:
                traffic = (json.load(fp).get(top) or {}).get("dram_bytes_per_launch")
        # the dominant kernel by device time (the persistent C-loop kernel) has no
        # streaming algorithmic byte count: it moves random 32 B sectors; report its
        # measured DRAM throughput (ncu capture of the heaviest launch, same config)
        dom = max(prof, key=lambda k: prof[k]["ms"])
        dominant = {"kernel": dom, "share_of_device_time": prof[dom]["ms"] / total_ms if total_ms else None}
        if os.path.exists(tpath) and cfg.name == "C4" and dims == cfg.dims:
            with open(tpath) as fp:
                ent = json.load(fp).get(dom) or {}
            if ent:
                dur = float(ent["duration"].split()[0]) * {"ms": 1e-3, "us": 1e-6, "s": 1.0}[ent["duration"].split()[1]]
                gbs = ent["dram_bytes_per_launch"] / dur / 1e9
                dominant.update({"bound": "hbm (random 32 B sectors)", "dram_GBps_ncu": gbs,
                                 "frac_of_peak": gbs / peak, "source": "profiles/ncu_traffic_c4.json"})
        # random-access view (profiles/r02_random_gather_peak.json): a scattered
        # 4-byte access moves ~128 B of DRAM traffic on this B200, and random
        # reads saturate at ~37.8 G accesses/s; the graded kernel's DRAM traffic
        # (ncu) / bytes-per-access / its launch time against that ceiling
        random_access = None
        rpath = os.path.join(ROOT, "profiles", "r02_random_gather_peak.json")
        if traffic and os.path.exists(rpath):
            with open(rpath) as fp:
                rp = json.load(fp)
            bpa = statistics.mean(v for k, v in rp["ncu_dram_bytes_per_access"].items() if ", 0>" in k)
            acc_s = traffic / bpa / (per_launch_ms * 1e-3)
            random_access = {"achieved_Gaccess_s": acc_s / 1e9,
                             "peak_Gaccess_s": rp["random_read_ceiling_Gaccess_s"],
                             "frac": acc_s / 1e9 / rp["random_read_ceiling_Gaccess_s"],
                             "dram_bytes_per_access": bpa,
                             "source": "profiles/r02_random_gather_peak.json (tools/random_gather_peak.cu)"}
        roofline = {"kernel": top, "bound": "hbm", "achieved": achieved, "peak": peak,
                    "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                    "dram_over_algorithmic": (traffic / bytes_per_launch) if traffic else None,
                    "random_access": random_access,
                    "peak_source": peak_src,
                    "alg_bytes_per_launch": bytes_per_launch,
                    "mean_launch_us": per_launch_ms * 1e3,
                    "timed_launches": t_launch,
                    "share_of_device_time": prof[top]["ms"] / total_ms if total_ms else None,
                    "dominant_kernel": dominant,
                    "per_class_source": "one fully profiled warm-up step (every launch timed)",
                    "per_class": {k: {"launches_per_step": v["launches"],
                                      "ms_per_step": v["ms"],
                                      "achieved_GBps": v["achieved_GBps"],
                                      "frac": v["achieved_GBps"] / peak} for k, v in graded.items()}}

    # ---- verification report of the corrected field, device-resident
    verify = None
    if not sharded:
        g = dfh.clone()
        g[d_idx[:count]] = d_val[:count]
        torch.cuda.synchronize()
        vopts = P.DeriveOptions(device=dist.local)
        P.build_report_device(topo, df.data_ptr(), g.data_ptr(), xi, dtype, count, 0, vopts,
                              stream.cuda_stream)  # warm
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        flush.fill_(1.0)
        a.record(stream)
        rep = P.build_report_device(topo, df.data_ptr(), g.data_ptr(), xi, dtype, count, 0, vopts,
                                    stream.cuda_stream)
        b.record(stream)
        b.synchronize()
        del g
        vms = a.elapsed_time(b)
        verify = {"ms": vms, "value": n / (vms * 1e-3) / 1e6, "unit": UNIT,
                  "api": "mssz_cu_verify_device (build_report, tools/mssz.cpp:84-104)",
                  "passed": rep.passed(), "mss_distortion": rep.mss_distortion, "psnr": rep.psnr,
                  "bound_violations": rep.bound_violations, "edit_ratio": rep.edit_ratio,
                  "false_extrema": [rep.fp_max, rep.fp_min, rep.fn_max, rep.fn_min],
                  "gpu_launches": rep.kernel_launches}

    # ---- base codec on the GPU: the reconstruction producing fhat
    base_codec = None
    if not sharded and f is not None:
        tc, td = {}, {}
        recon, sym, lits = P.compress_base(topo, f, xi, tc)
        back = P.decompress_base(topo, sym, lits, xi, dtype, td)
        base_codec = {"compress_device_ms": tc["device_ms"], "decompress_device_ms": td["device_ms"],
                      "decompress_value": n / (td["device_ms"] * 1e-3) / 1e6, "unit": UNIT,
                      "escapes": int(lits.size),
                      "identical_to_input_fhat": bool(recon.tobytes() == fh.tobytes()),
                      "round_trip": bool(back.tobytes() == recon.tobytes()),
                      "api": "mssz_cu_compress_base / mssz_cu_decompress_base (block wavefront)"}
        del recon, sym, lits, back

    # ---- edit-set encoding of this EditSet, store backend:
    # the GPU stages (delta, LEB128, RLE, histogram, bit packing) are timed
    edit_codec = None
    if not sharded:
        es_host = P.EditSet(d_idx[:count].cpu().numpy().astype(np.uint64), d_val[:count].cpu().numpy())
        tm = {}
        t0 = time.perf_counter()
        payload = P.encode_edits(es_host, 0, tm)
        wall = time.perf_counter() - t0
        edit_codec = {"edits": int(count), "payload_bytes": len(payload), "device_ms": tm["device_ms"],
                      "wall_ms": wall * 1e3, "codec": "store",
                      "api": "mssz_cu_encode_edits (byte-identical to encode_edits, edit_codec.cpp:188-222)"}
        del es_host, payload

    # ---- e2e through the host API with pinned buffers
    e2e = None
    if not args.no_e2e:
        hf = (df.cpu() if sharded else torch.from_numpy(f)).pin_memory()
        hfh = (dfh.cpu() if sharded else torch.from_numpy(fh)).pin_memory()
        h_idx = torch.empty(max(count, 1), dtype=torch.int64).pin_memory()
        h_val = torch.empty(max(count, 1), dtype=tdtype).pin_memory()
        e2e_opts = P.DeriveOptions(subloop_cap=cfg.subloop_cap, device=dist.local)

        def host_step():
            if comm is not None:
                c, _, _ = comm.derive_edits_into(dims, hf.data_ptr(), hfh.data_ptr(), xi,
                                                 h_idx.data_ptr(), h_val.data_ptr(),
                                                 h_idx.numel(), dtype, e2e_opts)
                return c
            c, _ = P.derive_edits_into(topo, hf.data_ptr(), hfh.data_ptr(), xi, h_idx.data_ptr(),
                                       h_val.data_ptr(), h_idx.numel(), dtype, e2e_opts)
            return c

        host_step()
        walls = []
        dist.barrier()
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t = time.perf_counter()
            c2 = host_step()
            walls.append(time.perf_counter() - t)
        wall = dist.max(statistics.mean(walls))
        api = ("mssz_cu_derive_edits_slab (pinned host windows)" if sharded
               else "mssz_cu_derive_edits_into (pinned host buffers)")
        e2e = {"value": total_vertices / wall / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(dist.sum(2.0 * n_local * es)),
               "d2h_bytes_per_step": int(dist.sum(float(c2) * (8 + es))),
               "ms_per_step": wall * 1e3, "api": api}

    # ---- CPU baseline: the unmodified reference on a bounded sample (rank 0, N=1)
    cpu = None
    if not args.no_cpu and dist.rank == 0 and dist.world == 1:
        sdims = dims_arg(args.cpu_dims) or CPU_SAMPLE.get(cfg.name, cfg.dims)
        threads = os.cpu_count() or 1
        os.environ.setdefault("OMP_WAIT_POLICY", "active")
        try:
            times, cst, inputs, ref_res = cpu_reference_run(cfg, sdims, dtype, threads, steps=1,
                                                            want_inputs=True)
            sn = int(np.prod(sdims))
            cpu = {"value": sn / times[0] / 1e6, "unit": UNIT, "cores": threads,
                   "kind": "reference",
                   "sample": f"derive_edits on {cfg.kind} {'x'.join(map(str, sdims))} "
                             f"({sn} vertices), rel {cfg.rel}, {times[0]:.2f} s",
                   "same_config": list(sdims) == list(dims),
                   "edit_stats": cst,
                   "same_input": same_input_comparison(P, cfg, sdims, inputs, ref_res, times[0],
                                                       dist.local)}
            del inputs, ref_res
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    st = stats[-1]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": cfg.note, "dims": list(dims), "vertices": n, "kind": cfg.kind,
                   "rel_eb": cfg.rel, "xi": xi, "subloop_cap": cfg.subloop_cap,
                   "parallelism": (f"z-slab x{dist.world} (NCCL)" if sharded
                                   else f"replica-per-gpu x{dist.world}"),
                   "l2": "flushed between steps (512 MB write outside the timed events)",
                   "input_gen_s": round(t_gen, 2)},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "verify": verify,
        "base_codec": base_codec,
        "edit_codec": edit_codec,
        "gpu_launches": int(dist.sum(float(sum(s.kernel_launches for s in stats)))),
        "clocks": clk,
        "edit_stats": {"outer_iterations": st.outer_iterations, "c_passes": st.c_passes,
                       "sub_iterations": st.sub_iterations, "r_iterations": st.r_iterations,
                       "effective_edits": st.effective_edits, "touched": st.touched,
                       "label_passes": st.label_passes, "label_rounds": st.label_rounds,
                       "detect_sweeps": st.detect_sweeps,
                       "frontier_vertices": st.frontier_vertices,
                       "big_batches": st.big_batches, "huge_batches": st.huge_batches},
        "kernel_profile_ms_per_step": prof,
    }
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    dist.done()


if __name__ == "__main__":
    main()
