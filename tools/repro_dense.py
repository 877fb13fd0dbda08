import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2003_01216_b200 import _build
which = sys.argv[1]
N = 1 << 22
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
core = 5 * 10**17 + rng.integers(0, 10**6, N // 2)
keys = rng.permutation(np.concatenate([core, rng.integers(0, 10**18, N - N // 2)])).astype(np.int64)
lib = ctypes.CDLL(_build.SO_DEBUG if which == "debug" else _build.SO)
vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
lib.hs_sort.argtypes = [vp, i64, ci, ci, ci, vp]
d = torch.from_numpy(keys).cuda()
st = torch.cuda.current_stream().cuda_stream
if which == "plan":
    import paper_2003_01216_b200 as hs
    print(hs.hs_sort_plan(d, 18, 8))
    sys.exit(0)
rc = lib.hs_sort(d.data_ptr(), N, 1, 18, 8, st)
lib.hs_last_error_message.restype = ctypes.c_char_p
print("rc", rc, lib.hs_last_error_message(), flush=True)
torch.cuda.synchronize()
ok = np.array_equal(d.cpu().numpy(), np.sort(keys))
print("ok", ok)
