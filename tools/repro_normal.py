"""Dev repro: hs_sort (debug or product library via ctypes) on 2^22 normal(5e8, 2e7) int32 keys."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2003_01216_b200 import _build
lib = ctypes.CDLL(_build.SO_DEBUG if sys.argv[1] == "debug" else _build.SO)
vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
lib.hs_sort.argtypes = [vp, i64, ci, ci, ci, vp]
lib.hs_last_error_message.restype = ctypes.c_char_p
N = 1 << 22
keys = np.clip(np.random.default_rng(0).normal(5e8, 2e7, N), 0, 10**9 - 1).astype(np.int32)
d = torch.from_numpy(keys).cuda()
rc = lib.hs_sort(d.data_ptr(), N, 0, 9, 8, torch.cuda.current_stream().cuda_stream)
print("rc", rc, lib.hs_last_error_message(), flush=True)
torch.cuda.synchronize()
print("ok", np.array_equal(d.cpu().numpy(), np.sort(keys)))
