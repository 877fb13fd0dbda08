"""The debug library (-DHS_DEBUG: device-side invariant checks on shared-memory
indices, piece geometry and scatter positions -- standing in for
compute-sanitizer, which is closed on this pool) runs every entry point on a
spread of small inputs bit-exact, with no assert firing.  Runs in a
subprocess because a fired __trap() leaves the process's CUDA context
unusable."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_debug_build_all_entry_points():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2003_01216_b200 import _build
    _build.build(debug=True)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "debug_driver.py")], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "no device assert fired" in r.stdout


def test_debug_library_exports():
    """CPU: the debug library builds and exports the same C ABI."""
    import ctypes
    from paper_2003_01216_b200 import _build
    import paper_2003_01216_b200 as hs
    lib = ctypes.CDLL(_build.build(debug=True))
    for sym in hs.EXPORTED_SYMBOLS:
        assert hasattr(lib, sym), sym
