"""Generator known answers and C <-> numpy twin agreement.

The generator is input plumbing shared by the oracle tests and the GPU tests;
it holds none of the method's arithmetic (workload/__init__.py).
"""
import numpy as np
import pytest

import workload as W

# SURVEY.md Appendix A, first 8 keys per config.
FIRST8 = {
    "C1": [566561, 745781, 971002, 444359, 444264, 762894, 877348, 523067],
    "C2": [591189734, 749149683, 595638081, 765419154, 311588687, 346622270, 726353614, 739087324],
    "C3": [113450342, 700293513, 612974682, 72866736, 216439108, 636222315, 135145858, 888718434],
    "C4": [324415546, 333120293, 301465432, 323579631, 330644049, 881906930, 846235820, 490503227],
    "C5": [386768045983934041, 752307015838223999, 232709165677461822, 99339411326602529,
           187960121702422236, 380608927618621532, 985563523859852729, 511101488728492136],
}
# Appendix A bucket counts and fingerprints (sum64, xor64, mix64).
KAT = {
    "C1": ([104610, 104628, 104662, 105231, 104383, 104944, 104446, 105373, 104770, 105529],
           0x0000007A34A7F104, 0x000000000006602A, 0x80C5B47024824697),
    "C2": ([1678603, 1678725, 1679718, 1676928, 1674888, 1678167, 1678517, 1678805, 1676805, 1676060],
           0x001DCC0131B44AC4, 0x0000000007B8D372, 0x5EEA3B73B1892985),
    "C3": ([26841881, 26853000, 26841624, 26840704, 26842856, 26836432, 26846565, 26850548, 26841837, 26840009],
           0x01DCD35F069B398E, 0x000000002BD98D40, 0x4F485397FB3952F8),
    "C4": ([1839204, 2260188, 25544065, 25640097, 1890929, 2009151, 1982283, 2020972, 1982008, 1939967],
           0x0055865A9859671E, 0x0000000036AA195A, 0xCDD208C492479BBF),
    "C5": ([53686274, 53680909, 53686712, 53705206, 53688595, 53682215, 53682929, 53682733, 53687358, 53687981],
           0x5BFA775517BC26ED, 0x0FC0AE608BB7763D, 0xB15EDC6F4CD1C451),
}


def test_splitmix_seed0():
    # splitmix64 from state 0, first output.
    assert W.splitmix_output(0, 0) == 0xE220A8397B1DCDAF
    assert int(W.out_np(0, np.array([0], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("name", list(FIRST8))
def test_first8(name):
    assert W.generate(name, 0, 8).tolist() == FIRST8[name]
    assert W.generate_np(name, 0, 8).tolist() == FIRST8[name]


@pytest.mark.parametrize("name", list(FIRST8))
def test_c_matches_numpy_twin_on_slices(name):
    cfg = W.CONFIGS[name]
    for start in (0, 12345, cfg.n - 5000):
        a = W.generate(name, start, 5000)
        b = W.generate_np(name, start, 5000)
        np.testing.assert_array_equal(a, b)


def test_mixture_table():
    assert W.mixture_table("C4")[:4].tolist() == [654396439, 78766743, 168700712, 252846368]


def test_mulhi_np_bigint():
    rng = np.random.default_rng(0)
    x = rng.integers(0, 2**63, size=200, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    for r in (100, 10**6, 10**9, 10**18, 2**64 - 1):
        got = W.mulhi_np(x, r)
        exp = [(int(v) * r) >> 64 for v in x]
        assert [int(v) for v in got] == exp


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_appendix_a_full(name):
    keys = W.generate(name)
    cfg = W.CONFIGS[name]
    counts, s, x, m = KAT[name]
    assert np.bincount(keys // 10 ** (cfg.num_digits - 1), minlength=10).tolist() == counts
    fp = W.fingerprint(keys)
    assert (fp["sum64"], fp["xor64"], fp["mix64"]) == (s, x, m)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_appendix_a_full_big(name):
    keys = W.generate(name)
    cfg = W.CONFIGS[name]
    counts, s, x, m = KAT[name]
    assert np.bincount(keys // 10 ** (cfg.num_digits - 1), minlength=10).tolist() == counts
    fp = W.fingerprint(keys)
    assert (fp["sum64"], fp["xor64"], fp["mix64"]) == (s, x, m)


def test_determinism():
    a = W.uniform(10000, 42, 1000)
    b = W.uniform(10000, 42, 1000)
    np.testing.assert_array_equal(a, b)
    assert not np.array_equal(a, W.uniform(10000, 43, 1000))
