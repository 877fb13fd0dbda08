"""Kernel-variant experiments (dev aid).

  python tools/exp.py build NAME "-DHS_MERGE_VT=8 ..."   # -> var/NAME/libhybridsort.so (here, no GPU)
  python tools/exp.py run NAME [NAME ...] [--cfg C3]    # on the GPU box: per-kernel device times

Per-kernel times come from the CUPTI kernel trace of torch.profiler (device
time of every launch), averaged over the timed repetitions.
"""
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(name, defs):
    from paper_2003_01216_b200 import _build
    out = os.path.join(ROOT, "var", name)
    os.makedirs(out, exist_ok=True)
    so = os.path.join(out, "libhybridsort.so")
    cmd = [_build._nvcc(), *_build.NVCC_FLAGS, *defs.split(), "-I", _build.INCLUDE, "-I", _build.CSRC, "-o", so,
           *_build.sources()]
    subprocess.check_call(cmd)
    print("built", so)


def run_merge1(name, cfg_name="C3", reps=5, chunks=2):
    """One merge level in isolation: hs_merge(c=2) of a chunk-sorted array."""
    import numpy as np
    import torch
    from torch.profiler import profile, ProfilerActivity
    import paper_2003_01216_b200 as hs
    import workload as W
    cfg = W.CONFIGS[cfg_name]
    # input prepared with torch only (one hs library per process): stable
    # partition by leading digit, then each bucket's chunks sorted
    keys = torch.from_numpy(W.generate(cfg_name)).cuda()
    d = torch.clamp(keys.to(torch.int64) // 10 ** (cfg.num_digits - 1), 0, 9)
    order = torch.sort(d, stable=True).indices
    x = keys[order].contiguous()
    cnt = torch.bincount(d, minlength=10).cpu().tolist()
    offl = [0]
    for c_ in cnt:
        offl.append(offl[-1] + c_)
    off = torch.tensor(offl, dtype=torch.int64, device="cuda")
    for b in range(10):
        m = offl[b + 1] - offl[b]
        q, r = divmod(m, chunks)
        st0 = offl[b]
        for i in range(chunks):
            ln = q + (1 if i < r else 0)
            if ln:
                x[st0:st0 + ln] = torch.sort(x[st0:st0 + ln]).values
            st0 += ln
    torch.cuda.synchronize()
    path = ROOT + "/paper_2003_01216_b200/libhybridsort.so" if name == "main" else os.path.join(ROOT, "var", name, "libhybridsort.so")
    lib = hs.load(path)
    out = torch.empty_like(x)
    dt = 0 if x.dtype == torch.int32 else 1
    st = torch.cuda.current_stream().cuda_stream
    def call():
        rc = lib.hs_merge(x.data_ptr(), out.data_ptr(), x.numel(), dt, off.data_ptr(), chunks, st)
        assert rc == 0
    call(); call(); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            call()
        torch.cuda.synchronize()
    per = defaultdict(float)
    for ev in prof.events():
        if ev.device_type.name == "CUDA" and "hs::" in ev.name:
            per[ev.name.split("(")[0].replace("void hs::", "")] += ev.device_time_total
    nbytes = 2 * x.numel() * x.element_size()
    for k in sorted(per, key=lambda k: -per[k]):
        t = per[k] / reps / 1000
        print(f"   [merge1 {name}] {k[:60]:60s} {t:8.3f} ms  ({nbytes / (t / 1e3) / 1e9:.0f} GB/s alg)")


def run(names, cfg_name="C3", reps=5):
    import numpy as np
    import torch
    from torch.profiler import profile, ProfilerActivity
    import paper_2003_01216_b200 as hs
    import workload as W
    cfg = W.CONFIGS[cfg_name]
    src = torch.from_numpy(W.generate(cfg_name)).cuda()
    buf = torch.empty_like(src)
    for name in names:
        path = ROOT + "/paper_2003_01216_b200/libhybridsort.so" if name == "main" else os.path.join(ROOT, "var", name, "libhybridsort.so")
        lib = hs.load(path)
        dt = 0 if src.dtype == torch.int32 else 1
        stream = torch.cuda.current_stream().cuda_stream

        tags = torch.arange(buf.numel(), dtype=torch.int64, device=buf.device)

        def call():
            if os.environ.get("EXP_PAIRS"):
                rc = lib.hs_sort_pairs64(buf.data_ptr(), tags.data_ptr(), buf.numel(), cfg.num_digits, cfg.chunks,
                                         stream)
            else:
                rc = lib.hs_sort(buf.data_ptr(), buf.numel(), dt, cfg.num_digits, cfg.chunks, stream)
            assert rc == 0, lib.hs_last_error_message()
        for _ in range(2):
            buf.copy_(src); call()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps):
            buf.copy_(src)
            torch.cuda.synchronize()
            s.record(); call(); e.record(); torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ok = bool(torch.all(buf[1:] >= buf[:-1]))
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(reps):
                buf.copy_(src)
                call()
            torch.cuda.synchronize()
        per = defaultdict(float)
        cnt = defaultdict(int)
        for ev in prof.events():
            if ev.device_type.name == "CUDA" and "hs::" in ev.name:
                key = ev.name.split("(")[0].replace("void hs::", "")
                per[key] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
                cnt[key] += 1
        print(f"== {name} {cfg_name}: sort median {np.median(ts):.3f} ms ({cfg.n / np.median(ts) / 1e6:.2f} Gkeys/s) sorted={ok}")
        for k in sorted(per, key=lambda k: -per[k]):
            print(f"   {k[:70]:70s} {per[k] / reps / 1000:8.3f} ms/call  ({cnt[k] // reps} launches)")
        sys.stdout.flush()


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
    elif sys.argv[1] == "one":
        run([sys.argv[2]], sys.argv[3])
    elif sys.argv[1] == "merge1":
        for name in sys.argv[2:]:
            subprocess.call([sys.executable, __file__, "merge1one", name])
    elif sys.argv[1] == "merge1one":
        run_merge1(sys.argv[2])
    else:
        args = sys.argv[2:]
        cfg = "C3"
        if "--cfg" in args:
            i = args.index("--cfg"); cfg = args[i + 1]; args = args[:i] + args[i + 2:]
        for name in args:  # one process per variant (one static cudart per process)
            subprocess.call([sys.executable, __file__, "one", name, cfg])
