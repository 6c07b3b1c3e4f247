"""`orcasim._kernels` for the one reference test that calls a kernel directly
(test_lp.py: shuffle_into against the pure-Python shuffle_order): the device's shuffle through
the C ABI (orca_shuffle_order). Test infrastructure only."""
import ctypes as C

import numpy as np

from paper_2008_11578_b200._lib import check, load, ptr

FEASIBLE, FALLBACK_USED = 0, 1


def shuffle_into(perm, count, seed):
    """perm[:count] = the insertion order of `count` constraints under `seed` (_kernels.py:64-67)."""
    if count <= 0:
        return
    out = np.empty(int(count), dtype=np.int64)
    check(load().orca_shuffle_order(0, int(count), C.c_uint64(int(seed) & ((1 << 64) - 1)), ptr(out)))
    perm[:count] = out
