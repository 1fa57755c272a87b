"""Noise-rate variants of a compiled sampler without recompiling (test / bench tooling).

A compiled sampler's tensors do not depend on the noise rate -- only its error
model does (compile.cpp:172-180: reduce_channels over the same f images). The
full compile of the config-3 cultivation circuit takes most of an hour, so the
noise-rate sweep (bench.py --noise-scale) rescales the error model of the
committed p = 1e-3 model instead: every error outcome's probability is
multiplied by r = p'/p (a single mechanism's p, a joint table's entries o > 0)
and a joint table's no-error entry becomes 1 - sum(rest). This is the first-
order (in p) error model at p'; the channel merges of reduce_channels make the
exact model at p' differ at O(p'^2). It is a different, valid model -- the
reference's sampler loads and samples it like any other (parity tests run on
it), it is just not bit-identical to compiling the circuit at p'.

usage: python tools/noise_scale.py IN.zxs[.gz] r OUT.zxs
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_01059_b200 import zxs_format  # noqa: E402


def scale(arrays: dict, r: float) -> dict:
    out = {k: np.array(v, copy=True) for k, v in arrays.items()}
    p = out["mech_probability"]
    tb = out["mech_table_begin"]
    tab = out["table"]
    for m in range(len(tb) - 1):
        t0, t1 = int(tb[m]), int(tb[m + 1])
        if t1 > t0:  # joint: entry 0 = no flip (bit i of the index <-> f_vectors[i])
            tab[t0 + 1:t1] *= r
            rest = float(tab[t0 + 1:t1].sum())
            if rest > 1.0:
                raise ValueError(f"noise scale {r} makes mechanism {m} exceed probability 1")
            tab[t0] = 1.0 - rest
        else:
            p[m] = min(1.0, p[m] * r)
    return out


def main():
    src, r, dst = sys.argv[1], float(sys.argv[2]), sys.argv[3]
    zxs_format.save(dst, scale(zxs_format.load(src), r))


if __name__ == "__main__":
    main()
