"""Synthetic circuit generators for the BASELINE.json configs (test tooling).

There is no stim and no network here, so the benchmark circuits are
regenerated from their textbook definitions:

* rotated surface-code memory (configs 1, 2, 5) with uniform circuit-level
  depolarizing noise, optional T gate on one data qubit after RX;
* the [[19,1,5]] triangular 6.6.6 colour code memory with R_Z(theta)
  rotations on k data qubits (config 4);
* d=3 magic-state cultivation on the Steane colour code with circuit-level
  noise (config 3; Gidney et al.'s exact circuit is not available offline,
  the structure is reconstructed: `cultivation_d3`), and the round-1 Steane
  proxy (corrected checks);
* random small circuits in the spirit of tests/test_util.hpp:13-115.

Every generator is checked noiselessly by tests/test_circuits.py: the
reference's exact oracle (oracle.cpp:494) where the circuit is small enough,
otherwise the reference's exact P(all outputs 0 | no error).
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


# ---------------------------------------------------------------- cultivation
# Steane [[7,1,3]] colour code, Hamming labels 1..7 -> qubits 0..6; the three
# faces (weight-4 stabilisers, both X and Z type) are {4567}, {2367}, {1357}.
STEANE_FACES = [[3, 4, 5, 6], [1, 2, 5, 6], [0, 2, 4, 6]]
# Unitary encoder of the state on label 3 (qubit 2): X3 -> X3 X5 X6 (weight-3
# logical X), then pivots 4, 2, 1 (qubits 3, 1, 0, in |+>) fan out over their
# faces; qubits 4, 5, 6 start in |0>.
STEANE_ENCODER = [(2, 4), (2, 5), (3, 4), (3, 5), (3, 6), (1, 2), (1, 5), (1, 6), (0, 2), (0, 4), (0, 6)]


def steane_cultivation_proxy(checks: int, p: float) -> str:
    """Round-1 proxy, corrected: T-state injection into the
    Steane code, `checks` transversal H_XY checks (T on all data, RX anc,
    CX anc->q for all data, MX anc, T_DAG on all data, DETECTOR), final T on
    all data and MX of all data with observable = XOR of the 7. Noise only
    after encoding, on the check CX and before each ancilla readout.

    The round-1 version checked with T_DAG ... T, which measures a logical
    operator the T state is not an eigenstate of (both detectors were coin
    flips) and read the data out without the final T (a random observable).
    tests/test_circuits.py checks every generator noiselessly."""
    lines = ["RX 2", "T 2", "R 4 5 6", "RX 3 1 0"]
    lines += [f"CX {a} {b}" for a, b in STEANE_ENCODER]
    lines.append(f"DEPOLARIZE1({_fmt(p)}) 0 1 2 3 4 5 6")
    anc = 7
    for _ in range(checks):
        lines.append("T 0 1 2 3 4 5 6")
        lines.append(f"RX {anc}")
        for q in range(7):
            lines.append(f"CX {anc} {q}")
            lines.append(f"DEPOLARIZE2({_fmt(p)}) {anc} {q}")
        lines.append("T_DAG 0 1 2 3 4 5 6")
        lines.append(f"Z_ERROR({_fmt(p)}) {anc}")
        lines.append(f"MX {anc}")
        lines.append("DETECTOR rec[-1]")
    lines.append("T 0 1 2 3 4 5 6")
    lines.append("MX 0 1 2 3 4 5 6")
    lines.append("OBSERVABLE_INCLUDE(0) " + " ".join(f"rec[{-1 - i}]" for i in range(7)))
    return "\n".join(lines) + "\n"


def cultivation_d3(p: float, checks: int = 2, z_rounds: bool = True, round0: bool = True,
                   readout: str = "decode") -> str:
    """d=3 magic-state cultivation on the Steane colour code (the structure of
    Gidney, Shutty & Jones 2024, reconstructed offline) with circuit-level
    noise on every gate, reset and measurement:

    1. Injection: T|+> on qubit 2, unitary encoder into the colour code.
    2. Stabiliser round 0 (if round0): the three Z faces (R anc, CX q->anc,
       M anc) and the three X faces (RX anc, CX anc->q, MX anc) through one
       reused ancilla; every outcome is a detector (deterministic +1).
    3. `checks` H_XY double checks: T on all data; a Z-face round (z_rounds:
       detectors against the previous Z round -- Z faces commute with T, so
       they are measured inside the check frame); the transversal logical X
       measured through a fan-out from the ancilla (RX anc, CX anc->q x 7,
       MX anc, detector); T_DAG on all data.
    4. Readout ("decode"): the inverse encoder (noisy), M of qubits 4 5 6 and
       MX of qubits 3 1 0 (decoded stabilisers: detectors), T_DAG on qubit 2
       and MX (the logical T-basis readout: the observable). Readout "frame":
       T on all data and MX of all data, observable = XOR of the 7 (the H_XY
       value read in the check frame); the reference's simplifier then fuses
       the last check's T_DAG with that T, leaving chi = 432.

    Noise (p each): X_ERROR after R / Z_ERROR after RX, X_ERROR before M /
    Z_ERROR before MX, DEPOLARIZE2 after every CX, DEPOLARIZE1 on every T /
    T_DAG. A depolarizing channel commutes with any unitary on its qubit
    (D(U rho U^+) = U D(rho) U^+), so the T gates' channel sits after T and
    before T_DAG: the same noisy circuit, written so that the reference's
    simplifier (simplify.cpp:67-103) still fuses a check's T_DAG with the next
    check's T (an X-type error spider between them would block the fusion and
    take chi from 93,312 to ~1.5e9). No idle noise.

    Deterministic noiselessly: tests/test_circuits.py (the reference's exact
    oracle on reduced variants, and P(all zero | no error) = 1 on the full
    compiled circuit)."""
    L: list[str] = []
    nm = [0]
    rec: dict = {}
    anc = 7
    pf = _fmt(p)

    def meas(kind, q, key):
        if p:
            L.append(f"{'X' if kind == 'M' else 'Z'}_ERROR({pf}) {q}")
        L.append(f"{kind} {q}")
        rec[key] = nm[0]
        nm[0] += 1

    def det(keys):
        L.append("DETECTOR " + " ".join(f"rec[{rec[k] - nm[0]}]" for k in keys))

    def reset(kind, qs):
        L.append(f"{kind} " + " ".join(map(str, qs)))
        if p:
            L.append(f"{'X' if kind == 'R' else 'Z'}_ERROR({pf}) " + " ".join(map(str, qs)))

    def gate1(g, qs, noise_before=False):
        if p and noise_before:
            L.append(f"DEPOLARIZE1({pf}) " + " ".join(map(str, qs)))
        L.append(f"{g} " + " ".join(map(str, qs)))
        if p and not noise_before:
            L.append(f"DEPOLARIZE1({pf}) " + " ".join(map(str, qs)))

    def cx(a, b):
        L.append(f"CX {a} {b}")
        if p:
            L.append(f"DEPOLARIZE2({pf}) {a} {b}")

    D = list(range(7))
    reset("RX", [2])
    gate1("T", [2])
    reset("R", [4, 5, 6])
    reset("RX", [3, 1, 0])
    for a, b in STEANE_ENCODER:
        cx(a, b)
    zr = [0]

    def z_round():
        r = zr[0]
        for k, face in enumerate(STEANE_FACES):
            reset("R", [anc])
            for q in face:
                cx(q, anc)
            meas("M", anc, ("z", r, k))
            det([("z", r, k)] if r == 0 else [("z", r, k), ("z", r - 1, k)])
        zr[0] += 1

    if round0:
        z_round()
        for k, face in enumerate(STEANE_FACES):
            reset("RX", [anc])
            for q in face:
                cx(anc, q)
            meas("MX", anc, ("x", k))
            det([("x", k)])
    for c in range(checks):
        gate1("T", D)
        if z_rounds:
            z_round()
        reset("RX", [anc])
        for q in D:
            cx(anc, q)
        meas("MX", anc, ("c", c))
        det([("c", c)])
        gate1("T_DAG", D, noise_before=True)
    if readout == "frame":
        gate1("T", D)
        for q in D:
            meas("MX", q, ("d", q))
        L.append("OBSERVABLE_INCLUDE(0) " + " ".join(f"rec[{rec[('d', q)] - nm[0]}]" for q in D))
        return "\n".join(L) + "\n"
    for a, b in reversed(STEANE_ENCODER):
        cx(a, b)
    for q in (4, 5, 6):
        meas("M", q, ("d", q))
        det([("d", q)])
    for q in (3, 1, 0):
        meas("MX", q, ("d", q))
        det([("d", q)])
    gate1("T_DAG", [2], noise_before=True)
    meas("MX", 2, ("d", 2))
    L.append(f"OBSERVABLE_INCLUDE(0) rec[{rec[('d', 2)] - nm[0]}]")
    return "\n".join(L) + "\n"


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
