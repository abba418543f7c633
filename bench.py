"""Benchmark of the RIANN per-frame ANN-field query on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one frame of BASELINE.json's headline workload (config 3: 1080p RGB,
8x8x3 = 192-D patches, n = 65,536 references; 2,052,649 queries per frame).
Timed window: frames W+1 .. W+K of the seeded 60-frame clip (frame 1 starts
from init_field and is reported separately as `frame1`).  The frame's grid rows
are split into bands, one per rank (one process per GPU, NCCL); `--gpus N`
without torchrun re-launches itself under torch.distributed.run.  Rank 0
prints one JSON line.

  value     query patches/s with inputs resident in HBM (frames pre-uploaded,
            field and previous units device-resident), CUDA events on the
            library's stream, max over ranks.
  e2e       the same metric through the public API with host frames from
            pinned memory and the whole field read back to the host every
            frame: BandStream at N=1, DistributedStream (NCCL gather of the
            band fields to rank 0, device to device) at N>1.
  roofline  the query path (all its kernels in one frame) against measured
            HBM bandwidth: `traffic` = ncu DRAM bytes of the last timed frame,
            captured in-run by a child process under ncu (same inputs, same
            state), `achieved` = traffic / that frame's CUDA-event time.  The
            SURVEY §8d algorithmic figure is `effective_gbs` (it counts
            L2-served reference rows, so it can exceed HBM).
  cpu_baseline  the CPU oracle (C port of the reference, all host threads)
            on a bounded sample of positions; `busy_threads` is measured.
  configs   ms/frame of BASELINE configs 0-2 (whole clips) and the config-4
            exact comparator on one 4K frame (N=1 only).
--impl reference times the CPU port alone (rank 0; other ranks exit 0).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import resource
import shutil
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_1508_07953_b200 import workloads as W  # noqa: E402

NPH = 10  # RIANN_NPHASES
METRIC = "query patches/sec per ANNF (1080p RGB, 8x8x3 patches, n=65536)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--cpu-positions", type=int, default=512)
    ap.add_argument("--ref-positions", type=int, default=2048)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-comparator", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-ncu", action="store_true")
    ap.add_argument("--comparator-queries", type=int, default=262144)
    ap.add_argument("--ncu-child", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thr = threading.Thread(target=self._read, daemon=True)
            self.thr.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thr.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 9 for k in range(4)
                          if r[5 + k].lower() in ("active", "1")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic_bytes(st, dim, n):
    """SURVEY.md §8d per-frame bytes of the query path (frame read excluded):
    16 B/position (prev idx in, idx + f64 dist out) + 4 B per first-ring entry
    + 8*ceil(log2 n) B per ring (two binary searches) + 4*D B per distance."""
    return (16 * st.queries + 4 * st.first_ring_total + 8 * math.ceil(math.log2(n)) * st.total_rings
            + 4 * dim * st.total_distance_evals)


def sample_positions(gw, y0, y1, count, seed=1234):
    """Stratified seeded sample of grid positions inside rows [y0, y1)."""
    rng = np.random.default_rng(seed)
    rows = np.linspace(y0, y1 - 1, num=min(count, y1 - y0), dtype=np.int64)
    per = int(math.ceil(count / len(rows)))
    pos = []
    for y in rows:
        pos.extend(int(y) * gw + rng.choice(gw, size=per, replace=False))
    return np.array(sorted(set(pos))[:count], dtype=np.int64)


def sample_units(frame, cfg, pos, gw):
    from oracle import oracle as O

    raw = W.patch_rows(frame, cfg.patch, pos // gw, pos % gw)
    return O.normalize_rows(raw)[0]


class CpuMeter:
    """Process CPU time over a wall-clock interval -> busy host threads."""

    def __enter__(self):
        r = resource.getrusage(resource.RUSAGE_SELF)
        self.c0, self.t0 = r.ru_utime + r.ru_stime, time.perf_counter()
        return self

    def __exit__(self, *exc):
        r = resource.getrusage(resource.RUSAGE_SELF)
        self.cpu = r.ru_utime + r.ru_stime - self.c0
        self.wall = time.perf_counter() - self.t0

    @property
    def busy(self):
        return self.cpu / max(self.wall, 1e-9)


# ---------------------------------------------------------------------------
def run_reference(a):
    """--impl reference: the CPU port of the reference (oracle/, C, all host
    threads) on a bounded sample of positions; steps = frames."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O

    cfg = W.CONFIGS[a.config]
    gw, gh = cfg.grid
    K, Wm = a.steps, a.warmup
    frames = list(W.iter_clip(cfg, Wm + K))
    refs = W.reference_set(cfg)
    om = O.LazyOracleModel(refs) if cfg.n_refs > 8192 else O.OracleModel.build(refs)
    pos = sample_positions(gw, 0, gh, a.ref_positions)
    prev = O.init_field_indices(gw, gh, len(refs), 0).ravel()[pos]
    threads = os.cpu_count() or 1
    units = [sample_units(f, cfg, pos, gw) for f in frames]
    # pass 1 (untimed): the trajectory; builds every table row it touches
    # (the reference keeps its whole table in RAM; rows here are its preprocessing)
    t0 = time.perf_counter()
    prevs = [prev]
    for t in range(Wm + K):
        r = O.query_positions(om, units[t], prevs[-1], pos, gw, 0, t + 1, nthreads=threads)
        prevs.append(r["idx"])
    t_rows = time.perf_counter() - t0
    # pass 2: time each step (frame) on the warm model
    times, busy = [], []
    for t in range(Wm + K):
        with CpuMeter() as m:
            r = O.query_positions(om, units[t], prevs[t], pos, gw, 0, t + 1, nthreads=threads)
        times.append(m.wall)
        busy.append(m.busy)
        assert np.array_equal(r["idx"], prevs[t + 1])
    timed = times[Wm:]
    qps = len(pos) * K / sum(timed)
    line = {
        "metric": METRIC, "value": qps, "unit": "query patches/s", "impl": "reference",
        "n_gpus": world, "steps": K, "warmup": Wm, "ms_per_step": 1e3 * sum(timed) / K,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded blurred-noise clip, BASELINE config shape)",
        "config": {"workload": f"{cfg.name}: frames {Wm + 1}..{Wm + K}", "queries_per_frame": cfg.queries,
                   "sample_positions_per_step": int(len(pos)), "table_rows_built_s": t_rows},
        "cpu_baseline": {"value": qps, "unit": "query patches/s", "cores": threads, "kind": "port",
                         "busy_threads": float(np.mean(busy[Wm:])),
                         "sample": f"{len(pos)} stratified positions x {K} frames (after {Wm} warm-up "
                                   f"frames) of {cfg.name}; C port of search.py:83-151 in oracle/, "
                                   f"{threads} threads, chunks of ceil(positions / (4 threads))"},
        "e2e": {"value": qps, "unit": "query patches/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_comparator(R, N, ctx, model, frame, riann_idx, riann_dist, m):
    """K4 (evaluation.py:24-50 exact_nn) on m grid positions of one frame:
    device-resident unit rows, CUDA events on the library stream.  Reports the
    tensor roofline of the screen GEMM (algorithmic 2*m*n*D flops) and how often
    the RIANN field equals the exact nearest reference."""
    import torch

    units = R.frame_units(frame, model)
    Q = units.shape[0]
    sel = np.unique(np.linspace(0, Q - 1, min(m, Q)).astype(np.int64))
    q = torch.from_numpy(np.ascontiguousarray(units[sel])).cuda()
    m = q.shape[0]
    idx = torch.empty(m, dtype=torch.int32, device="cuda")
    dist = torch.empty(m, dtype=torch.float64, device="cuda")
    lib = N.lib()
    st = (C.c_uint64 * 2)()
    ext = torch.cuda.ExternalStream(ctx.stream)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    with ctx.lock:
        torch.cuda.synchronize()
        N.check(lib.riann_exact_nn_device(ctx.h, q.data_ptr(), m, idx.data_ptr(), dist.data_ptr(), st))
        ev0.record(ext)
        for _ in range(reps):
            N.check(lib.riann_exact_nn_device(ctx.h, q.data_ptr(), m, idx.data_ptr(), dist.data_ptr(), None))
        ev1.record(ext)
        ev1.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    gi = idx.cpu().numpy()
    gd = dist.cpu().numpy()
    tflops = 2.0 * m * model.n * model.dim / (ms / 1e3) / 1e12
    peak = bf16_peak()
    ri, rd = riann_idx[sel], riann_dist[sel]
    return {"kernel": "exact_tc_kernel (tcgen05 kind::f16 M=128 N=256, TMEM accumulators, TMA 128B swizzle) + "
                      "float64 re-check", "queries": int(m), "n_refs": int(model.n), "dim": int(model.dim),
            "ms": ms, "queries_per_s": m / ms * 1e3,
            "roofline": {"bound": "tensor", "achieved": tflops, "peak": peak, "unit": "TFLOP/s",
                         "frac": tflops / peak, "flops": "2*m*n*D (one fp16 dot product per pair)"},
            "rechecks_per_query": st[0] / m, "full_scan_queries": int(st[1]),
            "riann_equals_exact_frac": float(np.mean(ri == gi)),
            "riann_dist_over_exact_mean": float(np.mean(rd / np.maximum(gd, 1e-300)))}


def bf16_peak():
    pp = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        with open(pp) as f:
            pk = json.load(f)
        if pk.get("bf16_tflops"):
            return float(pk["bf16_tflops"])  # burst (a kernel timed alone); fp16 dense rate = bf16
    return 1640.2


def phase_names(N):
    return [N.lib().riann_phase_name(k).decode() for k in range(NPH)]


def device_frames_run(N, ctx, frames, y0, t_first, ev_pairs=None):
    """riann_process_frame on device-resident frames (device-resident field and
    units), returns per-frame FrameStatsC.  ev_pairs: per-frame CUDA events."""
    lib = N.lib()
    stats = []
    for k, f in enumerate(frames):
        st = N.FrameStatsC()
        if ev_pairs is not None:
            ev_pairs[k][0].record()
        N.check(lib.riann_process_frame(
            ctx.h, C.c_void_p(f.data_ptr()), f.shape[0], f.shape[1], f.shape[2] if f.dim() == 3 else 1, y0,
            None, 0, t_first + k, 20, 0.25, 8, N.F_DEVICE_PTRS | N.F_TEMPORAL | N.F_KEEP_UNITS,
            None, None, C.byref(st)))
        if ev_pairs is not None:
            ev_pairs[k][1].record()
        stats.append(st)
    return stats


def band_projection(R, N, model, cfg, frames, Wm, K, local, bands=(2, 4, 8)):
    """Per-GPU share of an N-GPU run measured on this GPU: grid-row band 0 of
    N (frame rows [0, gh/N + ph - 1)) through the same frames, device-resident,
    CUDA events.  The model is replicated in a real N-GPU run, so the band's
    ms/frame is the projected per-GPU frame time (only one GPU is available
    here)."""
    import torch

    from paper_1508_07953_b200.bands import BandStream, band_rows, frame_band

    gw, gh = cfg.grid
    ph = cfg.patch[1]
    ctx = N.context(local)
    ext = torch.cuda.ExternalStream(ctx.stream)
    out = {}
    for nb in bands:
        y0, y1 = band_rows(gh, nb, 0)
        bs = BandStream(model, gw, gh, y0, y1, R.SearchParams(), device=local)
        for k in range(Wm):
            bs.step(frame_band(frames[k], y0, y1, ph))
        dev = [torch.from_numpy(frame_band(frames[Wm + k], y0, y1, ph)).cuda() for k in range(K)]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ctx.lock:
            ctx.select(bs.slot)
            with torch.cuda.stream(ext):
                e0.record()
                device_frames_run(N, ctx, dev, y0, Wm + 1)
                e1.record()
        e1.synchronize()
        bs.close()
        ms = e0.elapsed_time(e1) / K
        out[f"gpus{nb}"] = {"band_rows": y1 - y0, "ms_per_frame_per_gpu": ms,
                            "projected_query_patches_per_s": cfg.queries / ms * 1e3}
    return out


def config_line(R, N, cfg_id, local):
    """Throughput of another BASELINE config on this GPU: every frame of the
    clip through the device-resident path (frames pre-uploaded), frame 1
    separately (random init field)."""
    import torch

    from paper_1508_07953_b200.bands import BandStream

    cfg = W.CONFIGS[cfg_id]
    clip = W.clip(cfg)
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
    ctx = N.context(local)
    with ctx.lock:
        R.model.resident(ctx, model)
    gw, gh = cfg.grid
    bs = BandStream(model, gw, gh, 0, gh)
    ext = torch.cuda.ExternalStream(ctx.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(ext):
        e0.record()
    bs.step(clip[0])
    with torch.cuda.stream(ext):
        e1.record()
    e1.synchronize()
    ms1 = e0.elapsed_time(e1)
    dev = [torch.from_numpy(np.ascontiguousarray(f)).cuda() for f in clip[1:]]
    torch.cuda.synchronize()
    with ctx.lock:
        ctx.select(bs.slot)
        with torch.cuda.stream(ext):
            e0.record()
            sts = device_frames_run(N, ctx, dev, 0, 2)
            e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / len(dev)
    bs.close()
    evals = sum(s.total_distance_evals for s in sts) / sum(s.queries for s in sts)
    return {"workload": cfg.name, "queries_per_frame": cfg.queries, "n_refs": cfg.n_refs, "dim": cfg.dim,
            "frames_timed": f"2..{cfg.frames}", "ms_per_frame": ms, "frames_per_s": 1e3 / ms,
            "query_patches_per_s": cfg.queries / ms * 1e3, "frame1_ms": ms1, "evals_per_query": evals}


def config4_line(R, N, local):
    """Config 4 (4K, n=262,144): the exact comparator field on one frame
    (RIANN tables at this n need 512 GiB: DESIGN.md 'Config 4')."""
    import torch

    cfg = W.CONFIGS[4]
    refs = W.reference_set(cfg)
    frame = next(W.iter_clip(cfg, 1))
    model = R.ReferenceModel.from_refs(refs, cfg.patch)
    R.field_exact_oracle(frame[:600, :600], model)  # warm-up: operands + TMA descriptors
    ctx = N.context(local)
    ext = torch.cuda.ExternalStream(ctx.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(ext):
        e0.record()
    R.field_exact_oracle(frame, model)
    with torch.cuda.stream(ext):
        e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    flops = 2.0 * cfg.queries * cfg.n_refs * cfg.dim
    return {"workload": cfg.name, "what": "field_exact_oracle (K4 tcgen05 screen + FP64 re-check), whole 4K frame "
                                          "incl. frame upload, units and field read-back",
            "queries_per_frame": cfg.queries, "n_refs": cfg.n_refs, "ms_per_frame": ms,
            "query_patches_per_s": cfg.queries / ms * 1e3,
            "tflops_effective": flops / (ms / 1e3) / 1e12, "tflops_frac": flops / (ms / 1e3) / 1e12 / bf16_peak()}


def ncu_frame_traffic(a):
    """Re-run this bench's setup in a child process under ncu and capture DRAM
    bytes + duration of every kernel of the last timed frame (NVTX range
    'riann_bench_frame').  Returns (per-kernel list, error string)."""
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    with tempfile.TemporaryDirectory() as td:
        log = os.path.join(td, "ncu.csv")
        cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
               "--clock-control", "none", "--cache-control", "none", "--nvtx", "--nvtx-include",
               "riann_bench_frame/", "--csv", "--log-file", log, sys.executable, os.path.abspath(__file__),
               "--ncu-child", "--steps", str(a.steps), "--warmup", str(a.warmup)]
        env = dict(os.environ)
        for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
            env.pop(k, None)
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
        except subprocess.TimeoutExpired:
            return None, "ncu child timed out"
        if r.returncode != 0 or not os.path.exists(log):
            return None, f"ncu child rc={r.returncode}: {(r.stderr or r.stdout)[-300:]}"
        import csv

        rows = [x for x in csv.reader(open(log)) if len(x) > 10]
    if not rows:
        return None, "ncu captured no kernels"
    h = rows[0]
    ik, im, iv, iid, iu = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                           h.index("ID"), h.index("Metric Unit"))
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
             "s": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1.0, "KB": 1e3, "MB": 1e6,
             "GB": 1e9}
    by, names = {}, {}
    for x in rows[1:]:
        i = int(x[iid])
        names[i] = x[ik]
        by.setdefault(i, {})[x[im]] = float(x[iv].replace(",", "")) * scale.get(x[iu], 1.0)
    out = []
    for i in sorted(by):
        m = by[i]
        out.append({"kernel": names[i], "ms": m.get("gpu__time_duration.sum", 0.0),
                    "dram_bytes": m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)})
    return out, None


def run_ncu_child(a):
    """Under ncu: the same inputs and state as the parent's last timed frame,
    that frame alone inside the NVTX range the parent filters on."""
    import torch

    import paper_1508_07953_b200 as R
    from paper_1508_07953_b200.bands import BandStream

    cfg = W.CONFIGS[a.config]
    frames = list(W.iter_clip(cfg, a.warmup + a.steps))
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
    gw, gh = cfg.grid
    bs = BandStream(model, gw, gh, 0, gh)
    for f in frames[:-1]:
        bs.step(f)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("riann_bench_frame")
    bs.step(frames[-1])
    torch.cuda.nvtx.range_pop()
    bs.close()


def kernel_group(name):
    for key, label in (("units_warp", "units"), ("units_tile", "units"), ("units_kernel", "units"), ("pw_tree", "tc_tree"),
                       ("proj_kernel", "projection"), ("bulk_p0a", "p0a"), ("bulk_p0_", "p0b"),
                       ("bulk_draw", "draw"), ("anchor_scan", "group"), ("bulk_scatter", "group"), ("bulk_compact", "group"),
                       ("bulk_window", "window"), ("bulk_filter", "filter"), ("bulk_final", "final"),
                       ("query_kernel", "query (K2)")):
        if key in name:
            return label
    return name[:40]


# ---------------------------------------------------------------------------
def run_ours(a):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        assert dist.get_world_size() == a.gpus
    import paper_1508_07953_b200 as R
    from paper_1508_07953_b200 import _native as N
    from paper_1508_07953_b200.bands import BandStream, DistributedStream, band_rows, frame_band

    R.set_device(local)
    lib = N.lib()
    cfg = W.CONFIGS[a.config]
    K, Wm = a.steps, a.warmup
    gw, gh = cfg.grid
    y0, y1 = band_rows(gh, world, rank)
    pw, ph = cfg.patch

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        return float(t.item())

    # ---- inputs: W warm-up + K timed frames; band rows in pinned host memory
    t0 = time.time()
    total = Wm + K
    full_frames = list(W.iter_clip(cfg, total))
    host = []
    for f in full_frames:
        band = frame_band(f, y0, y1, ph)
        pinned = torch.empty(band.shape, dtype=torch.float32, pin_memory=True)
        pinned.numpy()[...] = band
        host.append(pinned)
    if rank != 0 or world == 1:
        full_frames = full_frames if world == 1 else None
    refs = W.reference_set(cfg)
    t_data = time.time() - t0
    model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
    ctx = N.context(local)
    torch.cuda.synchronize()
    t0 = time.time()
    with ctx.lock:
        R.model.resident(ctx, model)  # K3 table build on the GPU
    t_tables = time.time() - t0
    dev_frames = [host[Wm + k].cuda(non_blocking=True) for k in range(K)]
    torch.cuda.synchronize()
    ext = torch.cuda.ExternalStream(ctx.stream)

    # ---- value leg: its own stream slot; warm-up through the public band API
    # (frame 1 from the random init field timed on its own), then the K frames
    # device-resident with CUDA events per frame on the library stream
    vs = BandStream(model, gw, gh, y0, y1, R.SearchParams(), device=local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_w = time.perf_counter()
    with torch.cuda.stream(ext):
        e0.record()
    vs.step(host[0].numpy())
    with torch.cuda.stream(ext):
        e1.record()
    e1.synchronize()
    frame1_wall = time.perf_counter() - t_w
    frame1_ms = allmax(e0.elapsed_time(e1))
    for k in range(1, Wm):
        vs.step(host[k].numpy())
    clocks = ClockSampler(local)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with ctx.lock:
        ctx.select(vs.slot)
        N.check(lib.riann_timing_enable(ctx.h, 1))
        barrier()
        torch.cuda.synchronize()
        with torch.cuda.stream(ext):
            stats = device_frames_run(N, ctx, dev_frames, y0, Wm + 1, evs)
        evs[-1][1].synchronize()
        barrier()
        per_frame = [b.elapsed_time(c) for b, c in evs]
        ms_value = allmax(evs[0][0].elapsed_time(evs[-1][1]) / K)
        ms3 = (C.c_double * 3)()
        nfr, nl = C.c_uint64(0), C.c_uint64(0)
        N.check(lib.riann_timing_read(ctx.h, ms3, C.byref(nfr), C.byref(nl)))
        phases = (C.c_double * NPH)()
        N.check(lib.riann_timing_phases(ctx.h, phases, NPH))
        phases_last = (C.c_double * NPH)()  # the frame the ncu pass captures
        N.check(lib.riann_timing_phases_frame(ctx.h, -1, phases_last, NPH))
        N.check(lib.riann_timing_enable(ctx.h, 0))
        vfield = np.empty((y1 - y0) * gw, np.int32)
        N.check(lib.riann_field_get(ctx.h, N.ptr(vfield), None, vfield.size))
    vs.close()

    # ---- e2e leg: public API, host frames in, whole field out
    if world == 1:
        es = BandStream(model, gw, gh, y0, y1, R.SearchParams(), device=local)
        outs = [(torch.empty((y1 - y0, gw), dtype=torch.int32, pin_memory=True).numpy(),
                 torch.empty((y1 - y0, gw), dtype=torch.float64, pin_memory=True).numpy()) for _ in range(2)]
        for k in range(Wm):
            es.step(host[k].numpy())
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(K):
            oi, od = outs[k & 1]
            last = es.step(host[Wm + k].numpy(), out_idx=oi, out_dist=od)
        t_e2e = time.perf_counter() - t0
        e2e_last = last[0].ravel().copy()
        es.close()
        d2h = int(cfg.queries * 12)
    else:
        ds = DistributedStream(model, gw, gh, R.SearchParams(), device=local)
        for k in range(Wm):
            ds.step(host[k].numpy())
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_fields = []
        for k in range(K):
            e2e_fields.append(ds.step(host[Wm + k].numpy()))
        t_e2e = time.perf_counter() - t0
        ds.close()
        e2e_last = e2e_fields[-1][0].indices[y0:y1].ravel().copy() if rank == 0 else None
        d2h = int(cfg.queries * 20)
    t_e2e = allmax(t_e2e)
    clk = clocks.stop()
    replay_identical = bool(np.array_equal(vfield, e2e_last)) if e2e_last is not None else None

    # ---- N>1: the N-band field must equal the 1-band field (rank 0, every timed frame)
    bands_identical = None
    if world > 1 and rank == 0:
        one = BandStream(model, gw, gh, 0, gh, R.SearchParams(), device=local)
        ok = True
        for k in range(total):
            idx, dst, _ = one.step(full_frames[k])
            if k >= Wm:
                f, _ = e2e_fields[k - Wm]
                ok &= np.array_equal(idx, f.indices) and np.array_equal(dst.view(np.uint64),
                                                                        f.distances.view(np.uint64))
        one.close()
        bands_identical = bool(ok)

    # ---- K4 exact comparator (tcgen05 screen + float64 re-check) on a sample of the last frame
    comp = None
    last_idx = last_dist = None
    if rank == 0 and world == 1:
        last_idx, last_dist = last[0].ravel(), last[1].ravel()
    if rank == 0 and world == 1 and not a.no_comparator:
        comp = run_comparator(R, N, ctx, model, host[Wm + K - 1].numpy(), last_idx, last_dist,
                              a.comparator_queries)

    q_total = cfg.queries
    value = q_total / (ms_value / 1e3)
    e2e = q_total * K / t_e2e

    from paper_1508_07953_b200.engine import FrameStats

    fstats = [FrameStats(int(s.total_rings), int(s.total_distance_evals), 0.0, 0.0, int(s.queries),
                         first_ring_total=int(s.sum_first_ring)) for s in stats]
    alg_bytes_last = allsum(algorithmic_bytes(fstats[-1], cfg.dim, cfg.n_refs))
    qpath_ms = allmax(ms3[1] / K)
    evals = allsum(sum(s.total_distance_evals for s in fstats)) / allsum(sum(s.queries for s in fstats))
    names = phase_names(N)
    phase_all = [allmax(phases[k] / K) for k in range(NPH)]  # every rank joins every collective
    phase_ms = {names[k].split(":")[1]: phase_all[k] for k in range(NPH) if phase_all[k] > 0}
    phase_last = {names[k].split(":")[1]: phases_last[k] for k in range(NPH) if phases_last[k] > 0}

    # ---- CPU baseline: oracle on a sample of the last frame (rank 0, N=1)
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        from oracle import oracle as O

        om = O.LazyOracleModel(refs) if cfg.n_refs > 8192 else O.OracleModel.build(refs)
        pos = sample_positions(gw, 0, gh, a.cpu_positions)
        fi = Wm + K - 1
        # the GPU field of frame fi-1 (the e2e leg's second-to-last output buffer)
        prev_idx = outs[(K - 2) & 1][0].ravel()[pos] if K >= 2 else None
        if prev_idx is not None:
            units = sample_units(full_frames[fi], cfg, pos, gw)
            threads = os.cpu_count() or 1
            t0 = time.perf_counter()
            r = O.query_positions(om, units, prev_idx, pos, gw, 0, fi + 1, nthreads=threads)
            t_cold = time.perf_counter() - t0
            with CpuMeter() as m:
                r = O.query_positions(om, units, prev_idx, pos, gw, 0, fi + 1, nthreads=threads)
            gi, gd = last_idx[pos], last_dist[pos]
            parity = {"positions": int(len(pos)), "frame": fi + 1,
                      "idx_equal_frac": float(np.mean(gi == r["idx"])),
                      "dist_bit_equal_frac": float(np.mean(gd.view(np.uint64) == r["dist"].view(np.uint64))),
                      "max_rel_dist_err": float(np.max(np.abs(gd - r["dist"]) / np.maximum(r["dist"], 1e-300)))}
            cpu = {"value": len(pos) / m.wall, "unit": "query patches/s", "cores": threads, "kind": "port",
                   "busy_threads": m.busy,
                   "sample": f"{len(pos)} stratified positions of frame {fi + 1} ({cfg.name}), GPU prev field; "
                             f"C port of search.py:83-151 (oracle/), table rows built lazily before timing "
                             f"(cold pass {t_cold:.1f}s)"}

    # ---- projected per-GPU frame time at N = 2 / 4 / 8 (band 0 of N on this GPU)
    projection = None
    if rank == 0 and world == 1 and not a.no_configs:
        projection = band_projection(R, N, model, cfg, full_frames, Wm, K, local)

    # ---- other BASELINE configs on this GPU (N=1)
    configs = None
    if rank == 0 and world == 1 and not a.no_configs:
        configs = {}
        for cid in (0, 1, 2):
            try:
                configs[f"cfg{cid}"] = config_line(R, N, cid, local)
            except Exception as e:  # reported, never fatal for the headline
                configs[f"cfg{cid}"] = {"error": repr(e)[:200]}
        try:
            configs["cfg4"] = config4_line(R, N, local)
        except Exception as e:
            configs["cfg4"] = {"error": repr(e)[:200]}

    # ---- roofline: ncu DRAM bytes of the last timed frame (child process)
    peak, peak_kind = measured_peaks()
    roof = {"bound": "hbm", "peak": peak, "unit": "GB/s", "peak_kind": peak_kind,
            "kernel": "query path (every kernel of one frame from P0a to the final scan, incl. the projection "
                      "and K2 fallback on the side streams)",
            "frame_ms_live": per_frame[-1], "query_path_ms_live": qpath_ms,
            "effective_gbs": alg_bytes_last / (per_frame[-1] / 1e3) / 1e9,
            "effective_note": "SURVEY 8d algorithmic bytes (4*D per distance evaluation) / frame time; counts "
                              "L2-served reference rows, so it may exceed HBM"}
    kernels = None
    if rank == 0 and world == 1 and not a.no_ncu:
        launches, err = ncu_frame_traffic(a)
        if launches:
            qp = [x for x in launches if kernel_group(x["kernel"]) not in ("units", "tc_tree")]
            traffic = sum(x["dram_bytes"] for x in qp)
            frame_traffic = sum(x["dram_bytes"] for x in launches)
            achieved = frame_traffic / (per_frame[-1] / 1e3) / 1e9
            roof.update({"achieved": achieved, "frac": achieved / peak, "traffic": frame_traffic,
                         "traffic_query_path": traffic, "traffic_source":
                         "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (cache-control none) on the "
                         "last timed frame, re-run in a child process with the same inputs and state"})
            groups = {}
            for x in launches:
                g = groups.setdefault(kernel_group(x["kernel"]), {"launches": 0, "ncu_ms": 0.0, "dram_bytes": 0.0})
                g["launches"] += 1
                g["ncu_ms"] += x["ms"]
                g["dram_bytes"] += x["dram_bytes"]
            tot_ncu = sum(g["ncu_ms"] for g in groups.values())
            for name, g in groups.items():
                live = phase_last.get(name)  # the same frame as the ncu bytes
                g["ncu_share"] = g["ncu_ms"] / tot_ncu
                if live:
                    g["live_ms_same_frame"] = live
                    g["achieved_gbs"] = g["dram_bytes"] / (live / 1e3) / 1e9
                    g["frac"] = g["achieved_gbs"] / peak
            kernels = groups
        else:
            roof.update({"achieved": None, "frac": None, "traffic": None, "traffic_error": err})

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "query patches/s", "n_gpus": world, "steps": K,
            "warmup": Wm, "ms_per_step": ms_value, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded blurred-noise clip and reference crops with BASELINE config-3 shape)",
            "config": {"workload": f"{cfg.name}: {cfg.width}x{cfg.height}x{cfg.channels}, 8x8 patches, "
                                   f"n={cfg.n_refs}, L=20 alpha=0.25 max_rings=8; timed frames {Wm + 1}..{Wm + K} "
                                   f"of the 60-frame clip",
                       "queries_per_frame": q_total, "bands": world, "frames_per_s": 1e3 / ms_value,
                       "evals_per_query": evals,
                       "l2": "inputs larger than L2 (34 GB sorted tables, 1.6 GB unit rows per frame); "
                             "no flush", "table_build_s": t_tables, "data_gen_s": t_data},
            "frame1": {"ms_device": frame1_ms, "ms_wall_public_api": 1e3 * frame1_wall,
                       "note": "frame 1 starts from init_field (random prev): the heaviest frame"},
            "per_frame_ms": per_frame,
            "phases_ms_per_frame": phase_ms,
            "phases_ms_last_frame": phase_last,
            "roofline": roof,
            "kernels": kernels,
            "cpu_baseline": cpu,
            "parity": parity,
            "comparator": comp,
            "configs": configs,
            "multi_gpu_projection": projection,
            "e2e": {"value": e2e, "unit": "query patches/s", "ms_per_step": 1e3 * t_e2e / K,
                    "h2d_bytes_per_step": int(sum(h.numel() for h in host[:1]) * 4 * world),
                    "d2h_bytes_per_step": d2h,
                    "api": "bands.BandStream (N=1) / bands.DistributedStream (N>1, NCCL gather to rank 0)"},
            "gpu_launches": int(nl.value) * world,
            "replay_identical": replay_identical,
            "bands_identical_to_1band": bands_identical,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch_distributed(a):
    """--gpus N without torchrun: re-run this script under torch.distributed.run."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    raise SystemExit(subprocess.call(cmd))


def main():
    a = parse()
    if a.ncu_child:
        run_ncu_child(a)
    elif a.impl == "reference":
        run_reference(a)
    elif a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
