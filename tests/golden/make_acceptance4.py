"""Golden fixture for the reference's acceptance check #4 (randomized
eigensolver vs dense EVD, ref tests/acceptance.cpp:125-189).

The input matrix depends on libstdc++'s std::normal_distribution, so it is
built by the reference-side harness (oracle/_ref, ref_acceptance4_matrix:
the reference's RowMatrix / HouseholderQR through the eigen shim) and stored
with the reference's own eigs_sym results for seeds 1..50 (k=20, p=10, q=2):

  acceptance4.npz   g (500 x 500), dense (sorted |lambda| desc, positive
                    first), ref_vals (50 x 20), ref_resid (50)

Usage (build container, needs oracle/_ref): python tests/golden/make_acceptance4.py
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_bindings import RefLib  # noqa: E402


def main():
    ref = RefLib()
    n, k = 500, 20
    g = np.zeros((n, n))
    dense = np.zeros(n)
    fn = ref.lib.ref_acceptance4_matrix
    fn.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double)]
    fn.restype = None
    fn(g.ctypes.data_as(C.POINTER(C.c_double)), dense.ctypes.data_as(C.POINTER(C.c_double)))
    vals = np.zeros((50, k))
    resid = np.zeros(50)
    for s in range(1, 51):
        st, v, vecs, r = ref.eigs(g, k, 10, 2, s, threads=1)
        assert st == 0
        vals[s - 1] = v[:k]
        resid[s - 1] = r
    np.savez_compressed(HERE / "acceptance4.npz", g=g, dense=dense, ref_vals=vals,
                        ref_resid=resid)
    print("wrote acceptance4.npz")


if __name__ == "__main__":
    main()
