"""The hand-written device-wide primitives of the build path (kernels/prims.cuh):
radix sort, look-back scans and flagged selection against host restatements,
at sizes around the tile boundaries (scan tile 2048, selection tile 4096,
radix tile 8192) and at the sizes the configs sort (C5 root: 2^29 pairs on
27 key bits)."""
import ctypes as C

import pytest

from paper_2301_10841_b200._capi import check, lib

pytestmark = pytest.mark.gpu

SORT, SUM64, MAX32, SELECT, EXCL32 = range(5)


def run(engine, which, n, lo=0, hi=32, seed=1):
    bad = C.c_uint64(0)
    check(lib.fjg_device_primitive_check(engine._h, which, n, lo, hi, seed, C.byref(bad)))
    return bad.value


@pytest.mark.parametrize("n", [0, 1, 2, 31, 2047, 2048, 2049, 4095, 4096, 4097, 8191, 8192, 8193, 100003, 1 << 20])
@pytest.mark.parametrize("which", [SUM64, MAX32, SELECT, EXCL32])
def test_scans_and_select(engine, which, n):
    assert run(engine, which, n, seed=n + which) == 0


@pytest.mark.parametrize("n", [0, 1, 2, 100, 8191, 8192, 8193, 3 * 8192 + 5, 1000003])
@pytest.mark.parametrize("lo,hi", [(0, 1), (0, 9), (0, 16), (0, 27), (0, 32), (4, 20), (11, 27)])
def test_radix_sort(engine, n, lo, hi):
    """Stable, bits [lo, hi) only (1 to 4 passes; odd and even pass counts)."""
    assert run(engine, SORT, n, lo, hi, seed=n * 7 + lo + hi) == 0


def test_large(engine):
    """Sizes of the C5 build: the 2^29-row root sort and a 2^25-entry frontier scan."""
    assert run(engine, SORT, 1 << 29, 0, 27, seed=5) == 0
    assert run(engine, SUM64, 1 << 25, seed=6) == 0
    assert run(engine, SELECT, 1 << 28, seed=7) == 0
