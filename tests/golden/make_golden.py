"""Generate golden vectors from the UNMODIFIED reference headers.

Runs only in the build container (needs /root/reference): `make -C oracle ref` compiles
/root/reference/proj/include/stokesmg/*.hpp in place (through oracle/ref_shim, a minimal Eigen stand-in)
into oracle/_ref/libstokesmg_ref.so; this script calls it and writes tests/golden/fem1d_golden.json.
The committed JSON pins the CPU oracle (tests/test_oracle_golden.py) on machines without the reference.
"""
import ctypes
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "..", "..", "oracle", "_ref", "libstokesmg_ref.so")


def main():
    ref = ctypes.CDLL(LIB)
    ref.ref_default_penalty.restype = ctypes.c_double
    ref.ref_default_penalty.argtypes = [ctypes.c_int, ctypes.c_double]
    buf = np.zeros(1 << 16)
    r, c = ctypes.c_int(), ctypes.c_int()
    P = buf.ctypes.data_as(ctypes.c_void_p)

    def mat(fn, *args):
        rc = fn(*args, P, ctypes.c_int(buf.size), ctypes.byref(r), ctypes.byref(c))
        assert rc == 0
        return buf[: r.value * c.value].reshape(r.value, c.value).tolist()

    D = ctypes.c_double
    out = {"quadrature": [], "lobatto": [], "mass_1d": [], "derivative_1d": [], "sipg": [], "mass_dg": [],
           "mass_c0": [], "derivative_c0": [], "embedding": [], "penalty": [], "patches": []}
    for n in range(1, 10):
        p, w = np.zeros(n), np.zeros(n)
        ref.ref_gauss_quadrature(n, p.ctypes.data_as(ctypes.c_void_p), w.ctypes.data_as(ctypes.c_void_p))
        out["quadrature"].append({"n": n, "points": p.tolist(), "weights": w.tolist()})
    for n in range(2, 11):
        p = np.zeros(n)
        ref.ref_gauss_lobatto_points(n, p.ctypes.data_as(ctypes.c_void_p))
        out["lobatto"].append({"n": n, "points": p.tolist()})
    for k in range(1, 8):
        for h in (1.0, 0.5, 1.0 / 16):
            g = ref.ref_default_penalty(k, h)
            out["penalty"].append({"k": k, "h": h, "value": g})
            out["mass_1d"].append({"da": k, "dt": k, "h": h, "m": mat(ref.ref_mass_matrix_1d, k, k, D(h))})
            out["mass_1d"].append({"da": k + 1, "dt": k, "h": h, "m": mat(ref.ref_mass_matrix_1d, k + 1, k, D(h))})
            out["derivative_1d"].append({"dp": k, "dv": k + 1, "m": mat(ref.ref_derivative_matrix_1d, k, k + 1)})
            for cells in (1, 2, 4):
                out["sipg"].append({"degree": k + 1, "cells": cells, "h": h, "gamma": g, "left": 1, "right": 1,
                                    "m": mat(ref.ref_sipg_laplace_1d, k + 1, cells, D(h), D(g), 1, 1)})
                for left in (0, 2, 3):
                    for right in (0, 2, 3):
                        out["sipg"].append({"degree": k, "cells": cells, "h": h, "gamma": g, "left": left,
                                            "right": right,
                                            "m": mat(ref.ref_sipg_laplace_1d, k, cells, D(h), D(g), left, right)})
                out["mass_dg"].append({"degree": k, "cells": cells, "h": h,
                                       "m": mat(ref.ref_mass_matrix_dg, k, cells, D(h))})
                for drop in (0, 1):
                    out["mass_c0"].append({"degree": k + 1, "cells": cells, "h": h, "drop": drop,
                                           "m": mat(ref.ref_mass_matrix_c0, k + 1, cells, D(h), drop)})
                    if h == 1.0:
                        out["derivative_c0"].append({"pdeg": k, "cells": cells, "drop": drop,
                                                     "m": mat(ref.ref_derivative_matrix_c0, k, cells, drop)})
        for deg in (k, k + 1):
            for cont in (0, 1):
                out["embedding"].append({"degree": deg, "continuous": cont, "m": mat(ref.ref_embedding_1d, deg, cont)})
    for level in range(0, 3):
        cap = 10000
        vert = np.zeros(3 * cap, dtype=np.int32)
        cells = np.zeros(8 * cap, dtype=np.int64)
        color = np.zeros(cap, dtype=np.int32)
        n = ref.ref_enumerate_patches.__call__(3, 3, level, vert.ctypes.data_as(ctypes.c_void_p),
                                               cells.ctypes.data_as(ctypes.c_void_p),
                                               color.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(cap))
        out["patches"].append({"level": level, "vertex": vert[: 3 * n].tolist(), "cells": cells[: 8 * n].tolist(),
                               "color": color[:n].tolist()})
    with open(os.path.join(HERE, "fem1d_golden.json"), "w") as f:
        json.dump(out, f)
    print("wrote", os.path.join(HERE, "fem1d_golden.json"))


if __name__ == "__main__":
    main()
