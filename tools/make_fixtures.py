"""Generates tests/golden/: compiled samplers (.zxs) and golden outputs.

Runs in the container that has /root/reference (the oracle/_ref library is the
unmodified reference compiled in place). For every fixture circuit it writes

  circuits/<name>.stim            the circuit text
  tests/golden/<name>.zxs         compile_circuit output, flattened
  tests/golden/goldens.json       per fixture: compile info, and for fixed
                                  (seed, first_shot, shots): ones count and
                                  sha256 of the reference's column words from
                                  sample_detectors/measurements (sampler.cpp:306-320)
                                  and of sample_error_batch f-columns

Usage: python tools/make_fixtures.py [--only name,...] [--big]
(--big also compiles the config-3 cultivation circuit into data/: minutes and
~15 GB of host memory).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import circuits as C  # noqa: E402
from oracle import refdriver as R  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
CIRC = os.path.join(ROOT, "circuits")


def sha(cols: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(cols, np.uint64).tobytes()).hexdigest()


def ones(cols: np.ndarray) -> int:
    return int(np.unpackbits(np.ascontiguousarray(cols, np.uint64).view(np.uint8)).sum())


def fixtures():
    """(name, mode, text-or-None, sample plan) — plan: list of (seed, first_shot, shots)."""
    F = []
    read = lambda n: open(os.path.join(CIRC, n + ".stim")).read()  # noqa: E731
    big = [(1, 0, 1000), (1, 0, 100000), (2, 0, 1000), (7, 12345, 4097), (3, 2**32 - 96, 2000)]
    F.append(("c1_surface_d3_zmem", 0, read("c1_surface_d3_zmem"), big + [(1, 0, 1000000), (2, 0, 1000000)]))
    F.append(("c2_surface_d3_xmem_t", 0, read("c2_surface_d3_xmem_t"), big + [(1, 0, 1000000), (2, 0, 1000000)]))
    F.append(("c4_color_d5_rz3", 0, C.color_code_memory(6, 3, 1e-3, rz_count=3), big))
    F.append(("c5_surface_d7_r7", 0, C.surface_code_memory(7, 7, 1e-3, "Z"), [(1, 0, 1000), (5, 777, 20000)]))
    F.append(("surface_d3_xmem_rz5", 0, _rz5(), big[:4]))
    F.append(("surface_d3_xmem_9t", 0, _nine_t(), big[:4]))
    # f_width 122 > 63: the magic component reads its tensors through a component-local
    # parameter map on the monomial / deduplicated path
    F.append(("surface_d5_r5_xmem_rz3", 0, _rz_surface(5, 5, 3), big[:4]))
    small = [(1, 0, 1000), (9, 100, 777)]
    F.append(("h_t_h_m", 1, "H 0\nT 0\nH 0\nM 0\n", small))
    F.append(("bell_m", 1, "H 0\nCNOT 0 1\nM 0 1\n", small))
    F.append(("rx_t_mx_det", 0, "RX 0\nT 0\nMX 0\nDETECTOR rec[-1]\n", small))
    F.append(("oracle_mix_1", 0, "RX 0\nR 1\nR_Z(0.125) 0\nPAULI_CHANNEL_1(0.1, 0.1, 0.2) 0 1\n"
              "H 0\nCNOT 0 1\nDEPOLARIZE2(0.01) 0 1\nM 0 1\nDETECTOR rec[-1] rec[-2]\n", small))
    F.append(("oracle_mix_2", 0, "H 0\nT 0\nCNOT 0 1\nX_ERROR(0.2) 1\nM 0 1\n"
              "DETECTOR rec[-1] rec[-2]\nOBSERVABLE_INCLUDE(0) rec[-1]\n", small))
    F.append(("oracle_mix_3", 1, "MPP X0*Z1\nX_ERROR(0.25) 0\nM 0 1\n", small))
    F.append(("oracle_mix_4", 1, "R_Y(0.23) 0\nE(0.15) X0 Z1\nH 1\nM 0 1\n", small))
    F.append(("xerror_merge", 0, "X_ERROR(0.1) 0\nX_ERROR(0.2) 0\nM 0\nDETECTOR rec[-1]\n", small))
    F.append(("norm_sum", 1, "H 0\nT 0\nCNOT 0 1\nX_ERROR(0.2) 0\nZ_ERROR(0.1) 1\nM 0 1\n", small))
    F.append(("steane_inject", 0, C.steane_cultivation_proxy(0, 1e-3), small, True))  # cat5 plan: fixed front-end
    # the same circuit through the front-end as shipped (cat5 defect: wrong marginals, still a
    # sampler parity case; its heavy component exercises probability_of's global-tensor path)
    F.append(("steane_inject_shipped", 0, C.steane_cultivation_proxy(0, 1e-3), small, False))
    # config 3 with the check-frame readout (chi = 432, chain of 9, circuit-level noise): the
    # cultivation structure at a size the reference samples in seconds
    F.append(("c3_cultivation_d3_frame", 0, C.cultivation_d3(1e-3, readout="frame"), big[:4], True))
    # random circuits with magic (mixed component widths, R_Z/R_X, channels)
    import random
    rng = random.Random(20261017)
    k = 0
    while k < 24:
        text = C.random_circuit(rng, rng.randint(2, 4), rng.randint(8, 20), True, 0.3, 3, True)
        try:
            m = R.RefModel.compile(text, 0)
        except Exception:
            continue
        inf = m.info
        if inf["chi"] > 64 or inf["num_outputs"] == 0:
            continue
        F.append((f"random_{k:02d}", 0, text, small))
        k += 1
    return F


def _rz5() -> str:
    """d=3 X-memory + R_Z(0.1 pi) on 5 data qubits (SURVEY 'R_Z x5 proxy')."""
    t = C.surface_code_memory(3, 3, 1e-3, "X")
    lines = t.splitlines()
    data = lines[1].split()[1:]
    ins = [f"R_Z(0.1) {q}" for q in data[:5]]
    return "\n".join(lines[:3] + ins + lines[3:]) + "\n"


def _rz_surface(d: int, rounds: int, k: int) -> str:
    """d x d X-memory, `rounds` rounds, R_Z(0.1 pi) on the first k data qubits."""
    t = C.surface_code_memory(d, rounds, 1e-3, "X")
    lines = t.splitlines()
    data = lines[1].split()[1:]
    ins = [f"R_Z(0.1) {q}" for q in data[:k]]
    return "\n".join(lines[:3] + ins + lines[3:]) + "\n"


def _nine_t() -> str:
    """d=3 X-memory + T on all 9 data qubits (SURVEY '9-T proxy')."""
    t = C.surface_code_memory(3, 3, 1e-3, "X")
    lines = t.splitlines()
    data = lines[1].split()[1:]
    return "\n".join(lines[:3] + ["T " + " ".join(data)] + lines[3:]) + "\n"


def make(name, mode, text, plan, out_dir=GOLDEN, write_circuit=True, fixed=False, reuse=False):
    """fixed: compile with the front-end whose cat5 normalisation is fixed
    (oracle/Makefile `fixed`); sampling and goldens always use the unmodified
    reference library on the saved model."""
    if write_circuit:
        with open(os.path.join(CIRC, name + ".stim"), "w") as fp:
            fp.write(text)
    t0 = time.time()
    path = os.path.join(out_dir, name + ".zxs")
    if reuse and os.path.exists(path):  # an earlier (possibly interrupted) run already compiled it
        m = R.RefModel.load(path)
    else:
        m = R.RefModel.compile_fixed(text, mode) if fixed else R.RefModel.compile(text, mode)
        m.save(path)
    compile_s = time.time() - t0
    info = m.info
    if fixed or reuse:  # the .zxs round trip does not carry the compile stats: chi from the per-component chi
        from paper_2604_01059_b200 import zxs_format
        info["chi"] = int(np.prod(zxs_format.load(path)["comp_chi"].astype(np.float64)))
    rec = {"mode": mode, "info": info, "compile_s": round(compile_s, 3), "frontend": "fixed-cat5" if fixed else "reference",
           "circuit_sha256": hashlib.sha256(text.encode()).hexdigest(), "samples": [], "fcols": []}
    threads = os.cpu_count() or 8
    for seed, first, shots in plan:
        try:
            if first == 0:
                # the reference's public sampler; batches small enough that every host thread gets one
                bs = int(min(65536, max(64, -(-shots // threads) // 64 * 64)))
                cols = m.sample(shots, seed, batch_size=bs, threads=threads)
                src = "sample"
            else:
                raise ValueError
        except ValueError:
            cols = m.sample_rb(shots, seed, first_shot=first, batch_size=64, threads=threads)
            src = "run_batch"
        except RuntimeError as e:
            if "width mismatch" not in str(e):
                raise
            cols = m.sample_rb(shots, seed, first_shot=first, batch_size=64, threads=threads)
            src = "run_batch"
        rec["samples"].append({"seed": seed, "first_shot": first, "shots": shots, "ones": ones(cols),
                               "sha256": sha(cols), "source": src})
    for seed, first, shots in plan[:2]:
        f = m.sample_error_batch(min(shots, 4096), seed, first)
        rec["fcols"].append({"seed": seed, "first_shot": first, "shots": min(shots, 4096), "ones": ones(f),
                             "sha256": sha(f)})
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--big", action="store_true")
    args = ap.parse_args()
    os.makedirs(GOLDEN, exist_ok=True)
    gpath = os.path.join(GOLDEN, "goldens.json")
    goldens = json.load(open(gpath)) if os.path.exists(gpath) else {}
    only = set(filter(None, args.only.split(",")))
    for name, mode, text, plan, *fixed in fixtures():
        if only and name not in only:
            continue
        t = time.time()
        goldens[name] = make(name, mode, text, plan, fixed=bool(fixed and fixed[0]))
        print(f"{name}: {goldens[name]['info']['num_outputs']} outputs, chi={goldens[name]['info']['chi']}, "
              f"{time.time() - t:.1f}s", flush=True)
    goldens["_philox"] = [{"seed": s, "stream": st, "index": i, "u": R.uniform_at(s, st, i)}
                          for s, st, i in [(0, 0, 0), (1, 0, 0), (1, 5, 12345), (7, 0x80000000, 99),
                                           (2**64 - 1, 0xFFFFFFFF, 2**64 - 1), (123456789, 3, 2**32 + 5)]]
    with open(gpath, "w") as fp:
        json.dump(goldens, fp, indent=1, sort_keys=True)
    if args.big:
        # config 3: d=3 magic-state cultivation with circuit-level noise (tools/circuits.py
        # cultivation_d3), compiled by the front-end with the cat5 fix -- the unmodified
        # front-end's decomposition gives this circuit wrong marginals (tests/test_circuits.py)
        os.makedirs(os.path.join(ROOT, "data"), exist_ok=True)
        text = C.cultivation_d3(1e-3)
        t = time.time()
        rec = make("c3_cultivation_d3", 0, text, [(1, 0, 1024), (2, 1 << 20, 512)], out_dir=os.path.join(ROOT, "data"),
                   write_circuit=True, fixed=True, reuse=True)
        print(f"cultivation d=3: {rec['info']} {time.time() - t:.1f}s", flush=True)
        # 4 GB raw; xz -6 takes it to ~80 MB (zxs_format / refdriver read .zxs.xz)
        zp = os.path.join(ROOT, "data", "c3_cultivation_d3.zxs")
        import shutil
        import subprocess
        if shutil.which("xz"):
            subprocess.run(["xz", "-T0", "-6", "-f", zp], check=True)
        else:
            import lzma
            with open(zp, "rb") as src, lzma.open(zp + ".xz", "wb", preset=6) as dst:
                shutil.copyfileobj(src, dst, 1 << 24)
            os.remove(zp)
        with open(os.path.join(ROOT, "data", "c3_cultivation_d3.json"), "w") as fp:
            json.dump(rec, fp, indent=1)


if __name__ == "__main__":
    main()
