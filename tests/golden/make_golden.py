"""Generates tests/golden/*.npz from the UNMODIFIED reference engine.

Run in the build container (needs oracle/_ref, i.e. /root/reference at build
time):  python tests/golden/make_golden.py

For each body and each dims triple: compile_task on the reference preset /
statement text, make_task_data(seed=1, row-major, IntValued) — the reference's
own data generator (matrix.cpp:20-37, per-name seed engine.cpp:147) — then
run_naive (the reference's correctness oracle, naive.cpp:157-166) and also
run_adaptive (the reference's tiled executor); both results must agree
bit-for-bit before the fixture is written.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle as po  # noqa: E402

DIMS = [(64, 64, 64), (96, 128, 160), (257, 129, 65), (13, 17, 5), (32, 24, 40)]
SOURCES = {
    "gemm": ("matmul", None),
    "discount": ("q1", None),
    "boost": ("q2", None),
    "thrcount": ("q3", 100.0),
    "sqdiff": (po.SQDIFF_TEXT, None),
    "eqcount": (po.EQCOUNT_TEXT, None),
}


def main():
    for body, (src, tconst) in SOURCES.items():
        text = src if src.startswith("where") else po.preset_source(src)
        out = {}
        for (M, K, N) in DIMS:
            t = po.RefTask.create(text, M, K, N, seed=1, int_valued=True)
            assert t.is_mmlt()
            t.run_naive()
            naive = t.get("R").copy()
            t2 = po.RefTask.create(text, M, K, N, seed=1, int_valued=True)
            t2.run_adaptive()
            assert np.array_equal(naive, t2.get("R")), f"{body} {M}x{K}x{N}: adaptive != naive"
            key = f"{M}x{K}x{N}"
            out[key + "/A"] = t.get("A").astype(np.int8)
            out[key + "/B"] = t.get("B").astype(np.int8)
            if "thres" in t.names():
                out[key + "/thres"] = t.get("thres")[:, 0].astype(np.int8)
            if "dis" in t.names():
                out[key + "/dis"] = t.get("dis")[:, 0].astype(np.int8)
            out[key + "/R"] = naive
        meta = {"source": text, "thres_const": tconst if tconst is not None else np.nan}
        np.savez_compressed(os.path.join(HERE, f"{body}.npz"),
                            __source__=np.array(meta["source"]),
                            __thres_const__=np.array(meta["thres_const"]), **out)
        print("wrote", body, len(DIMS), "cases")


if __name__ == "__main__":
    main()
