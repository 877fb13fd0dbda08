#!/usr/bin/env python
"""bench.py -- Gkeys/s of the hybrid MSD-radix / merge sort hot path on B200.

One step = one hs_sort (C ABI, all kernels of the path: tile histograms,
lookback prefix, stable scatter, tile sort, merge levels) over one batch of
the BASELINE.json workload: C3 = 268,435,456 int32 keys uniform in [0, 1e9)
(seed 3, D = 9, 8 chunks per bucket), keys resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]
                  [--api sort|shared]

--api shared times hs_sort_shared instead (the no-MSD
ablation: chunk sort + tree merge of the whole array); --config P3 is
the paper's own 3-digit workload (f4).

N > 1 runs N independent replicas (one per GPU, launched by torchrun; the
path does not shard -- DESIGN.md §7), timed as the max over ranks.
--impl reference times the CPU oracle (oracle/, the plain C implementation
of the paper's algorithm) on bounded samples of the same workload.

Prints ONE JSON line on rank 0 (details on stderr).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gkeys/s end-to-end sort on 1 B200; per-kernel HBM GB/s vs peak"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload_desc(cfg):
    kind = ("uniform in [%d, %d)" % (cfg.value_lo, cfg.value_lo + cfg.value_range) if cfg.kind == "uniform"
            else "70/20/10 normal/1024-value/uniform mixture")
    return (f"{cfg.name}: {cfg.n:,} {cfg.dtype} keys, {kind}, seed {cfg.seed}, "
            f"D={cfg.num_digits} (MSD digit = floor(k/10^{cfg.num_digits - 1})), {cfg.chunks} chunks/bucket")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML while the timed region runs."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, torch_dev_index: int, period_s: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period_s
        self.ok = False
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            props = torch.cuda.get_device_properties(torch_dev_index)
            bus = "%08x:%02x:%02x.0" % (getattr(props, "pci_domain_id", 0), props.pci_bus_id, props.pci_device_id)
            try:
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(torch_dev_index)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # no NVML: report null clocks
            log(f"[bench] NVML unavailable: {e}")

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def result(self):
        if not self.ok or not self.samples:
            return None
        reasons = sorted(self.reasons - {"gpu_idle"})
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------- reference
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, cfg):
    """The base contract's reference arm, which for this paper is the CPU oracle (oracle/,
    plain C; its OpenMP build runs the paper's own shared-memory scheme on the box's host
    cores: chunks, then merge pairs, in parallel), timed as it stands on bounded samples."""
    import oracle
    import workload as W
    sample = min(cfg.n, args.ref_sample)
    nsteps = args.warmup + args.steps
    times = []
    threads = 1
    for i in range(nsteps):
        start = (i * sample) % max(cfg.n - sample + 1, 1)
        keys = W.generate(cfg, start, sample)
        _, dt, threads = oracle.timed_sort(keys, cfg.num_digits, cfg.chunks, openmp=True)
        if i >= args.warmup:
            times.append(dt)
    sec = statistics.mean(times)
    value = sample / sec / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "Gkeys/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype,
        "data": "synthetic",
        "config": {"workload": workload_desc(cfg), "sample_keys_per_step": sample,
                   "parallelism": f"host CPU, OpenMP oracle on {threads} threads ({cpu_model()})"},
        "cpu_baseline": {"value": value, "unit": "Gkeys/s", "cores": threads, "kind": "oracle",
                         "cpu": cpu_model(),
                         "sample": f"{sample:,} consecutive keys of {cfg.name} per step (bounded sample), "
                                   "OpenMP build of the plain C oracle (gcc -O2 -fopenmp; chunk quicksorts and "
                                   "merge pairs in parallel, P:58-62), time of the sort call only"},
        "e2e": {"value": value, "unit": "Gkeys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- ours
def cpu_baseline(cfg, sample, shared=False, sample_omp=None):
    """The oracle timed on this host, as it stands: its OpenMP build (the paper's shared-memory
    scheme on all host cores) on sample_omp keys -- the reported value -- and the plain
    single-thread build on `sample` keys beside it."""
    import oracle
    import workload as W
    ncores = host_cores()

    def one(nkeys, openmp):
        keys = W.generate(cfg, 0, nkeys)
        if shared:
            t0 = time.perf_counter()
            oracle.sort_shared(keys, cfg.chunks, openmp=openmp)
            dt = time.perf_counter() - t0
            thr = ncores if openmp else 1
        else:
            _, dt, thr = oracle.timed_sort(keys, cfg.num_digits, cfg.chunks, openmp=openmp)
        return nkeys / dt / 1e9, dt, thr

    n1 = sample
    v1, t1, _ = one(n1, False)
    single = {"value": v1, "unit": "Gkeys/s", "cores": 1, "kind": "oracle",
              "sample": f"first {n1:,} keys of {cfg.name} ({n1 / cfg.n:.3g} of the workload), plain single-thread "
                        f"C oracle (gcc -O2), {t1:.2f} s for the sort call only"}
    no = min(cfg.n, sample_omp or cfg.n)
    vo, to, thr = one(no, True)
    return {"value": vo, "unit": "Gkeys/s", "cores": thr, "kind": "oracle", "cpu": cpu_model(),
            "host_cores": ncores,
            "sample": f"first {no:,} keys of {cfg.name} ({no / cfg.n:.3g} of the workload), OpenMP build of the "
                      f"plain C oracle (gcc -O2 -fopenmp, {thr} threads: chunk quicksorts, then merge pairs, in "
                      f"parallel -- the paper's shared-memory scheme, P:58-62), {to:.2f} s for the sort call only",
            "single_core": single}


def run_ours(args, cfg):
    import numpy as np
    import torch
    import paper_2003_01216_b200 as hs
    import workload as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    hs.load()
    dt_code = 0 if cfg.dtype == "int32" else 1
    tdt = torch.int32 if cfg.dtype == "int32" else torch.int64
    ksize = 4 if cfg.dtype == "int32" else 8

    # inputs: generated on the host (seeded), pinned, copied once to HBM
    h_in = torch.empty(cfg.n, dtype=tdt, pin_memory=True)
    W.generate(cfg, 0, cfg.n, out=h_in.numpy())
    h_out = torch.empty_like(h_in, pin_memory=True)
    src = h_in.to(dev)
    buf = src.clone()  # (the graph's uncaptured warm-up call then sorts the real workload)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    shared = args.api == "shared"
    pairs = args.api == "pairs"
    if pairs:  # f3: int32 keys -> (key << 32 | index) items + tag gather; int64 keys -> the stable KV item path
        tags0 = torch.arange(cfg.n, dtype=torch.int64, device=dev)
        tags = torch.empty_like(tags0)

    graph = None
    if args.graph and (shared or pairs):
        raise SystemExit("--graph applies to hs_sort")
    if not (shared or pairs) and not args.no_graph:
        # the hs_sort call captured once in a CUDA graph (its ~33 launches and the
        # stream-ordered scratch allocation) and replayed every step: same kernels,
        # no per-launch host work (default; --no-graph times the direct call)
        graph = hs.SortGraph(buf, cfg.num_digits, cfg.chunks)

    def sort_step():
        if graph is not None:
            graph.replay()
        elif shared:
            hs.hs_sort_shared(buf, cfg.chunks)
        elif pairs:
            hs.hs_sort_pairs(buf, tags, cfg.num_digits, cfg.chunks)
        else:
            hs.hs_sort(buf, cfg.num_digits, cfg.chunks)

    def restore():
        buf.copy_(src)
        if pairs:
            tags.copy_(tags0)
        flush.fill_(1)

    for _ in range(args.warmup):
        restore()
        sort_step()
    torch.cuda.synchronize()
    ok = bool(torch.all(buf[1:] >= buf[:-1]).item())
    if not ok:
        raise SystemExit("[bench] hs_sort output is not sorted")
    if graph is not None:
        hs.hs_sort(buf, cfg.num_digits, cfg.chunks)  # launch count of one call (the graph replays them)
        torch.cuda.synchronize()
    launches_per_step = hs.last_launch_count()

    def barrier():
        if dist is not None:
            dist.barrier()

    # ---- timed region: K steps, CUDA events around each hs_sort
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    with sampler:
        for i in range(args.steps):
            restore()  # untimed: outside the event pair
            evs[i][0].record(stream)
            sort_step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    wall = time.perf_counter() - wall0
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = statistics.mean(step_ms)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * cfg.n / (ms * 1e-3) / 1e9

    # ---- per-kernel device times (library events on the launching stream)
    hs.profile_enable(True)
    for _ in range(args.steps):
        restore()
        if graph is not None:  # per-kernel events need the direct call (a replay records none)
            hs.hs_sort(buf, cfg.num_digits, cfg.chunks)
        else:
            sort_step()
    prof = hs.profile_read()
    hs.profile_enable(False)
    # algorithmic bytes of the dominant kernel from the plan of this workload
    if shared:  # one segment: the whole array is "bucket 0"
        off_h = np.array([0] + [cfg.n] * 10, dtype=np.int64)
    else:
        _, off = hs.hs_msd_partition(src, cfg.num_digits)
        off_h = off.cpu().numpy()
    kv = pairs and cfg.dtype == "int64"
    levels, tile_levels = hs.plan_levels(off_h, 1 if pairs else dt_code, cfg.chunks, 0)
    if kv:  # the item path's own tile capacity (no K5a split on it)
        t_kv, c = hs.tile_keys(1, 3), cfg.chunks
        levels = []
        for mm in np.diff(off_h).tolist():
            tiles = -(-(-(-mm // c)) // t_kv)  # ceil(ceil(m / c) / T)
            levels.append((int(tiles - 1).bit_length() if tiles > 1 else 0) + c.bit_length() - 1)
    split = [0] * 10
    if not shared and not pairs:  # the device plan: which buckets the K5a value split took
        dplan = hs.hs_sort_plan(src, cfg.num_digits, cfg.chunks)
        levels, split = dplan["levels"], dplan["split"]
    if pairs:
        ksize = 16 if kv else 8  # KV64 items, or (key << 32 | index) items through the int64 path
    m = np.diff(off_h)
    if pairs and not kv and prof.get("split_scatter", (0, 0))[1] > 0:  # int32 items: the int64 path's K5a split
        t64 = hs.tile_keys(1, 1)
        split = [int(-(-int(m[b]) // cfg.chunks) > t64) for b in range(10)]
        levels = [cfg.chunks.bit_length() - 1 if split[b] else levels[b] for b in range(10)]
    per_kernel = {}
    for kind, (tot, cnt) in prof.items():
        if cnt:
            per_kernel[kind] = {"ms_per_step": tot / args.steps, "launches_per_step": cnt // args.steps}
    dom = max(per_kernel, key=lambda k: per_kernel[k]["ms_per_step"])
    L_launch = per_kernel.get("merge_level", {}).get("launches_per_step", 0)
    level_bytes = [2 * ksize * int(sum(m[b] for b in range(10) if levels[b] > lv)) for lv in range(L_launch)]
    m_split = int(sum(m[b] for b in range(10) if split[b]))
    # the count pass reads only the split buckets that are not in the padded layout
    padded = dplan.get("padded", [0] * 10) if (not shared and not pairs) else [0] * 10
    m_count = int(sum(m[b] for b in range(10) if split[b] and not padded[b]))
    alg = {  # algorithmic bytes per step of each kernel kind
        "tile_hist": ksize * cfg.n, "scatter": 2 * ksize * cfg.n, "tile_sort": 2 * ksize * cfg.n,
        "merge_level": sum(level_bytes), "split_count": ksize * m_count, "split_scatter": 2 * ksize * m_split,
    }
    if pairs:  # K0 + K8: pack (r 4 + w 8) and unpack (r 8, tag gather 8, w 4 + 8); KV: r 8 + 8, w 16 and back
        alg["copy"] = cfg.n * (64 if kv else 40)
    for k, d in per_kernel.items():
        if k in alg and d["ms_per_step"] > 0:
            d["alg_GBps"] = alg[k] / (d["ms_per_step"] * 1e-3) / 1e9
    peak, peak_src = peaks()
    achieved = per_kernel[dom].get("alg_GBps")
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{cfg.name}.json")  # ncu capture of hs_sort on this config
    if os.path.exists(tp) and not (shared or pairs):
        with open(tp) as f:
            traffic = json.load(f).get(dom)
    active = [b for b in level_bytes if b > 0]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic, "peak_source": peak_src,
                "alg_bytes_per_launch": (statistics.mean(active) if dom == "merge_level" and active else alg.get(dom)),
                "launches_per_step": per_kernel[dom]["launches_per_step"],
                "active_launches_per_step": len(active) if dom == "merge_level" else 1}
    # hist r + scatter r/w (MSD path only) + K5a split count r + scatter r/w (split buckets) + tile sort r/w + merge levels
    path_bytes = ksize * cfg.n * (2 if shared else 5) + ksize * m_count + 2 * ksize * m_split + sum(level_bytes)
    if pairs and not kv:  # pack (r 4 + w 8), tag copy (r 8 + w 8), unpack (r 8 + tag gather 8 + w 4 + w 8)
        path_bytes += cfg.n * (12 + 16 + 28)
    elif kv:  # pack (r 8 + 8, w 16), unpack (r 16, w 8 + 8)
        path_bytes += cfg.n * (32 + 32)
    step_roof = {"alg_bytes_per_step": path_bytes, "bytes_per_key": path_bytes / cfg.n,
                 "t_roof_ms": path_bytes / (peak * 1e9) * 1e3,
                 "frac": path_bytes / (peak * 1e9) / (ms * 1e-3), "levels": max(levels),
                 "split_buckets": int(sum(split))}

    # ---- end to end through the public API with pinned host buffers
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        buf.copy_(h_in, non_blocking=True)
        sort_step()
        h_out.copy_(buf, non_blocking=True)
        b.record(stream)
        b.synchronize()
        if i >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
    e2e_serial = statistics.mean(e2e_ms)
    ok_e2e = bool(np.all(h_out.numpy()[1:] >= h_out.numpy()[:-1]))
    del buf  # the pipeline below holds its own three device slots

    # pipelined stream of batches through the public HostSortPipeline (hs_sort
    # API only): H2D of step i+1 and D2H of step i-1 overlap the sort of step i
    e2e_pipe_ms = None
    if not shared and not pairs:
        h_outs = [h_out, torch.empty_like(h_in, pin_memory=True)]
        pipe = hs.HostSortPipeline(cfg.n, tdt, cfg.num_digits, cfg.chunks, device=dev)
        for i in range(args.warmup):
            pipe.submit(h_in, h_outs[i & 1])
        pipe.finish()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(pipe.s_in)
        for i in range(args.steps):
            pipe.submit(h_in, h_outs[i & 1])
        pipe.s_out.wait_event(pipe.out_done[(args.steps - 1) & 1])
        b.record(pipe.s_out)
        pipe.finish()
        b.synchronize()
        e2e_pipe_ms = a.elapsed_time(b) / args.steps
        ok_e2e = ok_e2e and all(bool(np.all(h.numpy()[1:] >= h.numpy()[:-1])) for h in h_outs)
        del pipe
    e2e = e2e_pipe_ms if e2e_pipe_ms is not None else e2e_serial
    if dist is not None:
        t = torch.tensor([e2e, e2e_serial], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e, e2e_serial = float(t[0].item()), float(t[1].item())

    # context only: the library sort torch ships (a CUB radix sort that also returns
    # int64 indices) on the same device-resident keys, L2 flushed in between -- not a target
    context = None
    if world == 1 and not shared and not pairs and not args.no_context:
        x = src.clone()
        ts = []
        for i in range(2 + 5):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            torch.sort(x)
            b.record(stream)
            b.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b))
        del x
        tms = statistics.median(ts)
        context = {"torch_sort_ms": tms, "torch_sort_gkeys_s": cfg.n / (tms * 1e-3) / 1e9,
                   "note": "torch.sort (library radix sort; values + int64 indices) on the same keys; context only"}

    if rank == 0:
        log(f"[bench] {cfg.name} hs_sort {ms:.3f} ms/step = {value:.2f} Gkeys/s (steps {[round(x, 3) for x in step_ms]}), "
            f"wall {wall:.3f} s; e2e {e2e:.3f} ms/step pipelined, {e2e_serial:.3f} serial (sorted={ok_e2e})")
        for k, d in sorted(per_kernel.items(), key=lambda kv: -kv[1]["ms_per_step"]):
            log(f"[bench]   {k:16s} {d['ms_per_step']:8.3f} ms/step  {d['launches_per_step']:3d} launches  "
                f"{d.get('alg_GBps', 0):7.0f} GB/s alg")
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(cfg, min(cfg.n, args.cpu_sample), shared, args.cpu_sample_omp)
            log(f"[bench] cpu_baseline {cpu}")
        line = {
            "metric": METRIC, "value": value, "unit": "Gkeys/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "n_per_gpu": cfg.n, "num_digits": cfg.num_digits,
                       "api": ("hs_sort_shared (no MSD step, SURVEY f1)" if shared else
                               ("hs_sort_pairs64 (int64 key + 64-bit tag items on the stable KV path; SURVEY f3)" if kv
                                else "hs_sort_pairs (int32 key + 64-bit tag items, stable; SURVEY f3)") if pairs else
                               "hs_sort replayed from a CUDA graph (SortGraph)" if graph is not None else "hs_sort"),
                       "chunks_per_bucket": cfg.chunks, "merge_levels": max(levels),
                       "parallelism": "replicas" if world > 1 else "single GPU",
                       "l2": "flushed (256 MiB device write) before every timed step",
                       "timing": "mean of per-step CUDA-event intervals around hs_sort on the launching stream; "
                                 "the untimed input restore + L2 flush sit between the intervals; max over ranks"},
            "roofline": roofline,
            "path_roofline": step_roof,
            "kernels": per_kernel,
            "cpu_baseline": cpu,
            "e2e": {"value": world * cfg.n / (e2e * 1e-3) / 1e9, "unit": "Gkeys/s", "ms_per_step": e2e,
                    "h2d_bytes_per_step": cfg.n * ksize, "d2h_bytes_per_step": cfg.n * ksize,
                    "how": ("HostSortPipeline (public API): every step copies its batch pinned host -> device, "
                            "hs_sort, copies the sorted batch device -> pinned host; three device slots and three "
                            "streams overlap step i+1's H2D and step i-1's D2H with step i's sort; CUDA events "
                            "from the first H2D to the last D2H / K, max over ranks")
                    if e2e_pipe_ms is not None else
                    "pinned host keys -> H2D -> sort -> D2H, CUDA events on the stream, max over ranks",
                    "serial_ms_per_step": e2e_serial,
                    "serial_value": world * cfg.n / (e2e_serial * 1e-3) / 1e9},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": sampler.result(),
            "sorted_check": ok and ok_e2e,
            "context": context,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_dist(args, cfg):
    """the paper's cluster model over NCCL (weak scaling: every
    rank holds cfg.n keys of its own; one all-to-all-v moves each digit group
    to its owner rank, which sorts it).  Not the driver's default line."""
    import torch
    import torch.distributed as dist
    import paper_2003_01216_b200 as hs
    from paper_2003_01216_b200 import dist as hd
    import workload as W

    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29577")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = torch.device("cuda", local)
    hs.load()
    tdt = torch.int32 if cfg.dtype == "int32" else torch.int64
    h = torch.empty(cfg.n, dtype=tdt, pin_memory=True)
    W.generate(cfg, rank * cfg.n, cfg.n, out=h.numpy())
    src = h.to(dev)
    buf = src.clone()
    times = []
    info = None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    sampler = ClockSampler(local)

    def step():
        if args.fused:
            return hd.dist_sort_fused(buf, cfg.num_digits, cfg.chunks)
        return hd.dist_sort(buf, cfg.num_digits, cfg.chunks)

    with sampler:
        for i in range(args.warmup + args.steps):
            buf.copy_(src)
            flush.fill_(1)
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out, info = step()
            b.record()
            torch.cuda.synchronize()
            if i >= args.warmup:
                times.append(a.elapsed_time(b))
    launches = hs.last_launch_count()  # the local sort's kernels of the last step (plus K1-K3 on the fused path)
    ms = statistics.mean(times)
    # e2e: this rank's keys pinned host -> device, the distributed sort, its sorted piece device -> pinned host
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        buf.copy_(h, non_blocking=True)
        out, info = step()
        h_out = torch.empty(out.numel(), dtype=out.dtype, pin_memory=True)
        h_out.copy_(out, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
    t = torch.tensor([ms, statistics.mean(e2e_ms)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, e2e = float(t[0].item()), float(t[1].item())
    ok = bool(torch.all(out[1:] >= out[:-1]).item()) if out.numel() > 1 else True
    if rank == 0:
        line = {"metric": METRIC, "value": world * cfg.n / (ms * 1e-3) / 1e9, "unit": "Gkeys/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
                "config": {"workload": workload_desc(cfg) + f" per rank (keys [rank*n, (rank+1)*n) of the stream)",
                           "parallelism": (f"bucket sharding, exchange fused into the scatter (peer stores into "
                                           f"symmetric memory): {world} ranks (SURVEY f2, P:78-80)" if args.fused else
                                           f"bucket sharding over NCCL all-to-all-v: {world} ranks (SURVEY f2, P:78-80)"),
                           "group_start": info.group_start, "max_group_keys": info.max_load,
                           "l2": "flushed (256 MiB device write) before every timed step",
                           "timing": "CUDA events around dist_sort (partition, size all-gather, all-to-all-v, "
                                     "local hs_sort), max over ranks"},
                "e2e": {"value": world * cfg.n / (e2e * 1e-3) / 1e9, "unit": "Gkeys/s", "ms_per_step": e2e,
                        "h2d_bytes_per_step": world * cfg.n * h.element_size(),
                        "d2h_bytes_per_step": world * cfg.n * h.element_size(),
                        "how": "per rank: pinned H2D of its keys, the distributed sort, D2H of its sorted piece; "
                               "CUDA events, max over ranks"},
                "gpu_launches": launches * args.steps,
                "clocks": sampler.result(),
                "sorted_check": ok}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=1 << 26)
    ap.add_argument("--cpu-sample-omp", type=int, default=0, help="keys for the OpenMP oracle (0: the whole workload)")
    ap.add_argument("--ref-sample", type=int, default=1 << 25)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-context", action="store_true", help="skip the torch.sort context timing")
    ap.add_argument("--api", default="sort", choices=["sort", "shared", "pairs"])
    ap.add_argument("--dist", action="store_true", help="bucket-sharded multi-GPU sort (SURVEY f2)")
    ap.add_argument("--fused", action="store_true", help="with --dist: exchange fused into the scatter kernel")
    ap.add_argument("--graph", action="store_true", help="(default for --api sort) replay hs_sort from a CUDA graph")
    ap.add_argument("--no-graph", action="store_true", help="time direct hs_sort calls instead of a graph replay")
    args = ap.parse_args()
    import workload as W
    cfg = W.CONFIGS[args.config]
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        run_reference(args, cfg)
    elif args.dist:
        run_dist(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
