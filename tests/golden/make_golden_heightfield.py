"""Generate tests/golden/heightfield_ref.{abhf,csv} with the REFERENCE writers
(heightfield_io.cpp:30-45 / 86-103, compiled into oracle/_ref/libocean_ref.so).

Run here (where /root/reference exists):  python tests/golden/make_golden_heightfield.py
The input field is heightfield_input() below (also used by the tests), so the
files pin the byte layout of ABHF and the CSV number format.
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

OUT = os.path.dirname(os.path.abspath(__file__))
CASCADE, TIME = 3, 1.0 / 60.0


def heightfield_input(n=7):
    """Deterministic field with fp32-inexact values, signed zeros, tiny and large magnitudes."""
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    f = np.sin(0.7 * i + 1.3 * j) * 10.0 ** ((i - j) % 5 - 2) / 3.0
    f[0, 0], f[0, 1], f[1, 0] = 0.0, -0.0, 1e-40
    f[n - 1, n - 1] = -123456.789
    return f


def main():
    from oracle.oracle import build
    build(reference=True)
    L = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libocean_ref.so"))
    dp = C.POINTER(C.c_double)
    L.ref_write_heightfield.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_float, dp]
    L.ref_write_heightfield_csv.argtypes = [C.c_char_p, C.c_int, dp]
    f = np.ascontiguousarray(heightfield_input())
    n = f.shape[0]
    assert L.ref_write_heightfield(os.path.join(OUT, "heightfield_ref.abhf").encode(), n, CASCADE,
                                   TIME, f.ctypes.data_as(dp)) == 0
    assert L.ref_write_heightfield_csv(os.path.join(OUT, "heightfield_ref.csv").encode(), n,
                                       f.ctypes.data_as(dp)) == 0
    print("wrote heightfield_ref.abhf / .csv")


if __name__ == "__main__":
    main()
