"""Synthetic circuit generators for the BASELINE.json configs (test tooling).

There is no stim and no network here, so the benchmark circuits are
regenerated from their textbook definitions:

* rotated surface-code memory (configs 1, 2, 5) with uniform circuit-level
  depolarizing noise, optional T gate on one data qubit after RX;
* the [[19,1,5]] triangular 6.6.6 colour code memory with R_Z(theta)
  rotations on k data qubits (config 4);
* a Steane-code cultivation proxy: T injection, Clifford encoder and c
  transversal T checks (config 3 stand-in; Gidney et al.'s exact circuit
  is not available offline);
* random small circuits in the spirit of tests/test_util.hpp:13-115.

Every generator is validated by compiling it noiselessly with the reference
and checking that every detector and observable samples to 0.
"""
from __future__ import annotations

import random


def _fmt(x: float) -> str:
    return repr(float(x))


# ---------------------------------------------------------------- surface code
def surface_code_memory(d: int, rounds: int, p: float, basis: str = "Z", t_on_data: int | None = None) -> str:
    """Rotated surface code memory experiment, Stim-style layout: data at odd
    coordinates, measure qubits at even coordinates, X/Z CX orders
    xo=[(1,1),(1,-1),(-1,1),(-1,-1)], zo=[(1,1),(-1,1),(1,-1),(-1,-1)]."""
    assert basis in ("X", "Z") and d >= 2 and rounds >= 1
    data = [(2 * x + 1, 2 * y + 1) for x in range(d) for y in range(d)]
    xm, zm = [], []
    for x in range(d + 1):
        for y in range(d + 1):
            b1 = x == 0 or x == d
            b2 = y == 0 or y == d
            par = (x % 2) != (y % 2)
            if b1 and par:
                continue
            if b2 and not par:
                continue
            (xm if par else zm).append((2 * x, 2 * y))
    coords = sorted(set(data) | set(xm) | set(zm), key=lambda c: (c[1], c[0]))
    qid = {c: i for i, c in enumerate(coords)}
    D = [qid[c] for c in data]
    X = [qid[c] for c in xm]
    Z = [qid[c] for c in zm]
    anc = X + Z
    dset = set(data)
    xo = [(1, 1), (1, -1), (-1, 1), (-1, -1)]
    zo = [(1, 1), (-1, 1), (1, -1), (-1, -1)]

    def j(qs):
        return " ".join(str(q) for q in qs)

    lines = []
    if basis == "Z":
        lines.append(f"R {j(D + anc)}")
    else:
        lines.append(f"R {j(anc)}")
        lines.append(f"RX {j(D)}")
    lines.append(f"X_ERROR({_fmt(p)}) {j(D + anc)}")
    if t_on_data is not None:
        lines.append(f"T {D[t_on_data]}")
    nmeas = 0
    prev = None  # measurement index of each ancilla in the previous round
    for r in range(rounds):
        lines.append(f"DEPOLARIZE1({_fmt(p)}) {j(D)}")
        lines.append(f"H {j(X)}")
        lines.append(f"DEPOLARIZE1({_fmt(p)}) {j(X)}")
        for k in range(4):
            pairs = []
            for m in xm:
                dq = (m[0] + xo[k][0], m[1] + xo[k][1])
                if dq in dset:
                    pairs += [qid[m], qid[dq]]
            for m in zm:
                dq = (m[0] + zo[k][0], m[1] + zo[k][1])
                if dq in dset:
                    pairs += [qid[dq], qid[m]]
            lines.append(f"CX {j(pairs)}")
            lines.append(f"DEPOLARIZE2({_fmt(p)}) {j(pairs)}")
        lines.append(f"H {j(X)}")
        lines.append(f"DEPOLARIZE1({_fmt(p)}) {j(X)}")
        lines.append(f"X_ERROR({_fmt(p)}) {j(anc)}")
        lines.append(f"MR {j(anc)}")
        lines.append(f"X_ERROR({_fmt(p)}) {j(anc)}")
        cur = {a: nmeas + i for i, a in enumerate(anc)}
        nmeas += len(anc)
        for a in anc:
            if prev is None:
                if (basis == "Z" and a in Z) or (basis == "X" and a in X):
                    lines.append(f"DETECTOR rec[{cur[a] - nmeas}]")
            else:
                lines.append(f"DETECTOR rec[{cur[a] - nmeas}] rec[{prev[a] - nmeas}]")
        prev = cur
    lines.append(f"X_ERROR({_fmt(p)}) {j(D)}")
    lines.append(f"{'M' if basis == 'Z' else 'MX'} {j(D)}")
    dm = {q: nmeas + i for i, q in enumerate(D)}
    nmeas += len(D)
    checks = zm if basis == "Z" else xm
    order = zo if basis == "Z" else xo
    for m in checks:
        recs = [dm[qid[(m[0] + dx, m[1] + dy)]] - nmeas for dx, dy in order if (m[0] + dx, m[1] + dy) in dset]
        recs.append(prev[qid[m]] - nmeas)
        lines.append("DETECTOR " + " ".join(f"rec[{r}]" for r in recs))
    # logical: Z along a row (y = 1) for Z memory, X along a column (x = 1) for X memory
    line = [c for c in data if (c[1] == 1 if basis == "Z" else c[0] == 1)]
    lines.append("OBSERVABLE_INCLUDE(0) " + " ".join(f"rec[{dm[qid[c]] - nmeas}]" for c in line))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------- colour code
def _triangular_color_code(L: int):
    """6.6.6 triangular code from the triangular lattice:
    points (i+1, j), i, j >= 0, i + j <= L; colour (x - y) mod 3; colour-0
    points are face centres, others qubits; faces = hexagon neighbourhoods
    with >= 4 qubits in the patch."""
    pts = [(i + 1, j) for i in range(L + 1) for j in range(L + 1) if i + j <= L]
    qubits = [p for p in pts if (p[0] - p[1]) % 3 != 0]
    qs = set(qubits)
    nb = [(1, 0), (-1, 0), (0, 1), (0, -1), (1, -1), (-1, 1)]
    faces = []
    for p in pts:
        if (p[0] - p[1]) % 3 == 0:
            f = [q for q in ((p[0] + dx, p[1] + dy) for dx, dy in nb) if q in qs]
            if len(f) >= 4:
                faces.append(f)
    return qubits, faces


def color_code_memory(L: int, rounds: int, p: float, rz_count: int = 0, seed: int = 1) -> str:
    """X-memory on the triangular colour code (L=6 -> [[19,1,5]], L=3 ->
    Steane): separate X and Z ancilla per face, sequential CX, MX/M; X checks
    detected from round 1, Z checks from round 2; final MX of all data,
    observable = X on all data. R_Z(theta) (theta ~ U(0,1), units of pi,
    random.Random(seed)) on the first rz_count data qubits after RX."""
    qubits, faces = _triangular_color_code(L)
    nq = len(qubits)
    qi = {q: i for i, q in enumerate(qubits)}
    xa = [nq + 2 * k for k in range(len(faces))]
    za = [nq + 2 * k + 1 for k in range(len(faces))]
    D = list(range(nq))
    rng = random.Random(seed)

    def j(qs):
        return " ".join(str(q) for q in qs)

    lines = [f"R {j(xa + za)}", f"RX {j(D)}", f"DEPOLARIZE1({_fmt(p)}) {j(D)}"]
    for q in range(rz_count):
        lines.append(f"R_Z({_fmt(rng.random())}) {q}")
    nmeas = 0
    prev = None
    for r in range(rounds):
        lines.append(f"RX {j(xa)}")
        lines.append(f"R {j(za)}")
        for k, f in enumerate(faces):
            for q in f:
                lines.append(f"CX {xa[k]} {qi[q]}")
                lines.append(f"DEPOLARIZE2({_fmt(p)}) {xa[k]} {qi[q]}")
        for k, f in enumerate(faces):
            for q in f:
                lines.append(f"CX {qi[q]} {za[k]}")
                lines.append(f"DEPOLARIZE2({_fmt(p)}) {qi[q]} {za[k]}")
        lines.append(f"X_ERROR({_fmt(p)}) {j(za)}")
        lines.append(f"Z_ERROR({_fmt(p)}) {j(xa)}")
        lines.append(f"MX {j(xa)}")
        lines.append(f"M {j(za)}")
        cur = {a: nmeas + i for i, a in enumerate(xa + za)}
        nmeas += len(xa) + len(za)
        for a in xa + za:
            if prev is None:
                if a in xa:
                    lines.append(f"DETECTOR rec[{cur[a] - nmeas}]")
            else:
                lines.append(f"DETECTOR rec[{cur[a] - nmeas}] rec[{prev[a] - nmeas}]")
        prev = cur
        lines.append(f"DEPOLARIZE1({_fmt(p)}) {j(D)}")
    lines.append(f"Z_ERROR({_fmt(p)}) {j(D)}")
    lines.append(f"MX {j(D)}")
    dm = {q: nmeas + i for i, q in enumerate(D)}
    nmeas += nq
    for k, f in enumerate(faces):
        recs = [dm[qi[q]] - nmeas for q in f] + [prev[xa[k]] - nmeas]
        lines.append("DETECTOR " + " ".join(f"rec[{x}]" for x in recs))
    lines.append("OBSERVABLE_INCLUDE(0) " + " ".join(f"rec[{dm[q] - nmeas}]" for q in D))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------- cultivation proxy
def steane_cultivation_proxy(checks: int, p: float) -> str:
    """T-state injection into the Steane [[7,1,3]] code,
    `checks` transversal T checks (T_DAG on all data, RX anc, CX anc->q for
    all data, T on all data, MX anc, DETECTOR), final MX of all data with
    observable = XOR of the 7. Noise: DEPOLARIZE1 after encoding, DEPOLARIZE2
    on each check CX, Z_ERROR before each ancilla readout.

    Encoder (Hamming labels 1..7 -> qubits 0..6, stabilisers {4567}, {2367},
    {1357}): the state T|+> is prepared on label 3, copied to labels 5 and 6
    (X3 -> X3 X5 X6, a weight-3 logical X), then pivots 4, 2, 1 (in |+>)
    fan out over their stabilisers."""
    lines = ["RX 2", "T 2", "R 4 5 6", "RX 3 1 0", "CX 2 4 2 5",
             "CX 3 4 3 5 3 6", "CX 1 2 1 5 1 6", "CX 0 2 0 4 0 6"]
    lines.append(f"DEPOLARIZE1({_fmt(p)}) 0 1 2 3 4 5 6")
    anc = 7
    for _ in range(checks):
        lines.append("T_DAG 0 1 2 3 4 5 6")
        lines.append(f"RX {anc}")
        for q in range(7):
            lines.append(f"CX {anc} {q}")
            lines.append(f"DEPOLARIZE2({_fmt(p)}) {anc} {q}")
        lines.append("T 0 1 2 3 4 5 6")
        lines.append(f"Z_ERROR({_fmt(p)}) {anc}")
        lines.append(f"MX {anc}")
        lines.append("DETECTOR rec[-1]")
    lines.append("MX 0 1 2 3 4 5 6")
    lines.append("OBSERVABLE_INCLUDE(0) " + " ".join(f"rec[{-1 - i}]" for i in range(7)))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------- random circuits
def random_circuit(rng: random.Random, num_qubits: int, num_instructions: int, with_magic: bool,
                   max_p: float, max_channels: int, with_detectors: bool) -> str:
    """Random circuit over <= num_qubits qubits in the style of
    tests/test_util.hpp:23-112 (own generator; python RNG)."""
    out = []
    measurements = 0
    channels = 0

    def q():
        return rng.randint(0, num_qubits - 1)

    def pair():
        a, b = q(), q()
        if a == b:
            b = (a + 1) % num_qubits
        return a, b

    for _ in range(num_instructions):
        kind = rng.randint(0, 13 if with_magic else 9)
        if kind == 0:
            out.append(f"H {q()}")
        elif kind == 1:
            out.append(f"S {q()}")
        elif kind == 2:
            out.append(f"X {q()}")
        elif kind == 3:
            out.append(f"Z {q()}")
        elif kind == 4:
            out.append(f"SQRT_X {q()}")
        elif kind == 5:
            if num_qubits < 2:
                out.append(f"H {q()}")
            else:
                a, b = pair()
                out.append(f"{rng.choice(['CX', 'CZ'])} {a} {b}")
        elif kind == 6:
            if channels >= max_channels:
                out.append(f"S_DAG {q()}")
            else:
                channels += 1
                pp = rng.random() * max_p
                op = rng.choice(["X_ERROR", "Z_ERROR", "Y_ERROR", "DEPOLARIZE1"])
                out.append(f"{op}({_fmt(pp)}) {q()}")
        elif kind == 7:
            if channels >= max_channels or num_qubits < 2:
                out.append(f"H {q()}")
            else:
                channels += 1
                a, b = pair()
                out.append(f"DEPOLARIZE2({_fmt(rng.random() * max_p)}) {a} {b}")
        elif kind == 8:
            if measurements < 6:
                out.append(f"M {q()}")
                measurements += 1
            else:
                out.append(f"H {q()}")
        elif kind == 9:
            out.append(f"R {q()}")
        elif kind == 10:
            out.append(f"T {q()}")
        elif kind == 11:
            out.append(f"T_DAG {q()}")
        elif kind == 12:
            out.append(f"R_Z({_fmt(rng.random())}) {q()}")
        else:
            out.append(f"R_X({_fmt(rng.random())}) {q()}")
    if measurements == 0:
        out.append("M 0")
        measurements = 1
    if with_detectors:
        for _ in range(rng.randint(1, min(measurements, 3))):
            refs = " ".join(f"rec[-{rng.randint(1, measurements)}]" for _ in range(rng.randint(1, 2)))
            out.append(f"DETECTOR {refs}")
        out.append(f"OBSERVABLE_INCLUDE(0) rec[-{rng.randint(1, measurements)}]")
    return "\n".join(out) + "\n"


def noiseless(text: str) -> str:
    """Drops every noise channel (for determinism validation)."""
    keep = []
    for line in text.splitlines():
        head = line.split("(")[0].split(" ")[0]
        if head in ("X_ERROR", "Y_ERROR", "Z_ERROR", "DEPOLARIZE1", "DEPOLARIZE2", "PAULI_CHANNEL_1",
                    "PAULI_CHANNEL_2", "E", "CORRELATED_ERROR"):
            continue
        keep.append(line)
    return "\n".join(keep) + "\n"
