"""CPU emulation of the integer monomial path (mono_kernel) — no GPU needed.

zxs_debug_mono_layout returns the exact record streams and form dictionary
the device walks. This test decodes them the way mono_kernel does — per term
J (mod 4) and Z from the record kinds, epilogue Re(c' i^J) for non-zero
shots, terms in order — and checks the values against the C oracle's
eval_batch (phase_terms.cpp:90-144). The monomial path replaces the
reference's rounded h entries by their exact values, so agreement is to a
relative 1e-12 of the sum of |term| magnitudes (the reference's own rounding
is ~1e-16 per entry), not bit for bit.
"""
import ctypes

import numpy as np
import pytest

from conftest import golden_path
from oracle import coracle
from paper_2604_01059_b200 import _native, zxs_format

REC_ADD, REC_SUB, REC_ADD2, REC_Z, REC_ZN, REC_GEN = 0, 1, 2, 3, 4, 15
FORM_MASK, FORM_SHIFT_B = 0x3FFF, 14  # record word: kind << 28 | form b << 14 | form a (zxs_mono.cuh)


def mono_layout(arrays, min_factors=0):
    desc = zxs_format.make_desc(arrays)
    L = _native.lib()
    need = ctypes.c_uint64()
    _native.check(L.zxs_debug_mono_layout(ctypes.byref(desc), min_factors, None, 0, ctypes.byref(need)))
    buf = np.zeros(need.value, np.uint32)
    _native.check(L.zxs_debug_mono_layout(ctypes.byref(desc), min_factors,
                                          buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), buf.size,
                                          ctypes.byref(need)))
    n_words, n_chunks, n_tcb, n_dict, n_comps, n_components, all_plane = (int(x) for x in buf[:7])
    o = 8
    comps = [dict(zip(("ci", "n_out", "upos_base", "out_begin", "first_tensor"),
                      (int(v) for v in buf[o + 5 * i:o + 5 * i + 5]))) for i in range(n_comps)]
    o += 5 * n_comps
    flags = buf[o:o + n_components].astype(bool)
    o += n_components
    tcb = buf[o:o + n_tcb].astype(np.int64)
    o += n_tcb
    chunks = buf[o:o + 4 * n_chunks].reshape(n_chunks, 4).astype(np.int64)
    o += 4 * n_chunks
    dict_ = buf[o:o + 4 * n_dict].reshape(n_dict, 4).copy()
    o += 4 * n_dict
    tdb = buf[o:o + n_tcb].astype(np.int64)  # per mono tensor + total (same count as tcb)
    o += n_tcb
    twidth = buf[o:o + n_tcb - 1].astype(np.int64)
    o += n_tcb - 1
    tbb = buf[o:o + n_tcb - 1].astype(np.int64)
    o += n_tcb - 1
    nb = int(buf[o])
    o += 1
    basis = [int(buf[o + 2 * i]) | (int(buf[o + 2 * i + 1]) << 32) for i in range(nb)]
    o += 2 * nb
    words = buf[o:o + n_words]
    o += n_words
    n_tsb, n_segs, n_sw, n_km = (int(x) for x in buf[o:o + 4])
    o += 4
    tsb = buf[o:o + n_tsb].astype(np.int64)
    o += n_tsb
    segs = buf[o:o + 4 * n_segs].reshape(n_segs, 4).astype(np.int64)
    o += 4 * n_segs
    seg_words = buf[o:o + n_sw]
    o += n_sw
    key_mask = [int(buf[o + 2 * i]) | (int(buf[o + 2 * i + 1]) << 32) for i in range(n_km)]
    o += 2 * n_km
    n_tfb, n_bfb, n_bf = (int(x) for x in buf[o:o + 3])
    o += 3
    tfb = buf[o:o + n_tfb].astype(np.int64)
    o += n_tfb
    bfb = buf[o:o + n_bfb].astype(np.int64)
    o += n_bfb
    bforms = buf[o:o + n_bf].astype(np.int64)
    o += n_bf
    n_spw = int(buf[o])
    spw = buf[o + 1:o + 1 + n_spw].astype(np.int64)
    o += 1 + n_spw
    n_rm, n_nb, n_null = (int(x) for x in buf[o:o + 3])
    o += 3
    u64 = lambda a: [int(a[2 * i]) | (int(a[2 * i + 1]) << 32) for i in range(len(a) // 2)]  # noqa: E731
    read_mask = u64(buf[o:o + 2 * n_rm])
    o += 2 * n_rm
    null_begin = buf[o:o + n_nb].astype(np.int64)
    o += n_nb
    null = u64(buf[o:o + 2 * n_null])
    return dict(read_mask=read_mask, null_begin=null_begin, null=null, tfb=tfb, bfb=bfb, bforms=bforms, spw=spw, comps=comps, flags=flags, tcb=tcb, chunks=chunks, dict=dict_, tdb=tdb, twidth=twidth,
                tbb=tbb, basis=basis, all_plane=all_plane, words=words, tsb=tsb, segs=segs,
                seg_words=seg_words, key_mask=key_mask)


def form_sel(dict_, f):
    """Plane indices of dictionary form f (continuation entries followed):
    byte 0 = size class c (2c + 2 slots, 15 for c = 7) | 0x80, bytes 1..15 plane indices."""
    sel = []
    while True:
        e = dict_[f].view(np.uint8)
        slots = (2, 4, 6, 8, 10, 12, 14, 15)[int(e[0]) & 7]
        sel += [int(x) for x in e[1:1 + slots]]  # padding slots name the all-zero plane
        if not (int(e[0]) & 0x80):
            return sel
        f += 1


FV_FORM_BYTES = 128  # block form tables: a one-form record word is the form's byte offset (fv[form][lane])


def apply_node_records(w, q, h0, h1, h2, form, J, Z, block=False):
    """mono_kernel's one-form records (any kind order) and two-form records on (J, Z);
    returns the new position. block: dedup_eval_kernel's block-table segments, whose
    one-form records are grouped by kind (the header's counts) and hold fv byte offsets."""
    counts = (h1 & 0xFF, (h1 >> 8) & 0xFF, (h1 >> 16) & 0xFF, h1 >> 24, h2 & 0xFF)
    kinds = [k for k, n in zip((REC_ADD, REC_SUB, REC_ADD2, REC_Z, REC_ZN), counts) for _ in range(n)]
    for kind_by_pos in kinds:
        r = int(w[q])
        q += 1
        if block:
            assert r % FV_FORM_BYTES == 0
            kind, a = kind_by_pos, form(r // FV_FORM_BYTES)
        else:
            kind, a = r >> 28, form(r & FORM_MASK)
        if kind == REC_ADD:
            J += a
        elif kind == REC_SUB:
            J -= a
        elif kind == REC_ADD2:
            J += 2 * a
        elif kind == REC_Z:
            Z |= a == 1
        else:
            assert kind == REC_ZN
            Z |= a == 0
    for _ in range(h0 & 0xFF):
        r, g = int(w[q]), int(w[q + 1])
        q += 2
        assert r >> 28 == REC_GEN
        fa, fb = r & FORM_MASK, (r >> FORM_SHIFT_B) & FORM_MASK
        a = 0 if fa == FORM_MASK else form(fa)
        b = 0 if fb == FORM_MASK else form(fb)
        zl = g >> 6
        Z |= ((zl >> (a * 2 + b)) & 1) == 1
        J += (g & 3) * a + ((g >> 2) & 3) * b + ((g >> 4) & 3) * (a * b)
    return q


SEG_START = 1 << 30


def walk_nodes(w, nnodes, form, S, stack, acc, tot, stats=None, block=False):
    """mono_walk: nnodes nodes of stream w; FOLD when tot is given (segment starts
    fold the running sum into tot)."""
    q = 0
    for _ in range(nnodes):
        h0, h1, h2 = int(w[q]), int(w[q + 1]), int(w[q + 2])
        depth, leaf = (h0 >> 24) & 0x3F, h0 >> 31
        if tot is not None and h0 & SEG_START:
            tot += acc
            acc[:] = 0.0
        q += 3
        if leaf:
            re = w[q:q + 2].copy().view(np.float64)[0]
            im = w[q + 2:q + 4].copy().view(np.float64)[0]
            q += 4
        if depth:
            J, Z = stack[depth - 1][0].copy(), stack[depth - 1][1].copy()
        else:
            J, Z = np.zeros(S, np.int64), np.zeros(S, bool)
        q = apply_node_records(w, q, h0, h1, h2, form, J, Z, block)
        if stats is not None:
            stats["nodes"] = stats.get("nodes", 0) + 1
        if not leaf:
            stack[depth] = (J, Z)
            continue
        J &= 3
        v = np.where(J == 0, re, np.where(J == 1, -im, np.where(J == 2, -re, im)))
        acc[:] = np.where(Z, acc, acc + v)


def tensor_forms(lay, t, P):
    d0 = int(lay["tdb"][t])
    W = int(lay["twidth"][t])
    planes = np.zeros((P.shape[0], lay["all_plane"] + 2), np.int64)
    b0 = int(lay["tbb"][t])
    for b in range(W):
        m = lay["basis"][b0 + b]
        cols = [p for p in range(64) if (m >> p) & 1]
        planes[:, b] = P[:, cols].sum(1) & 1 if cols else 0
    planes[:, lay["all_plane"]] = planes[:, :W].sum(1) & 1
    cache = {}

    def form(f):
        if f not in cache:
            cache[f] = (planes[:, form_sel(lay["dict"], d0 + f)].sum(1) & 1).astype(np.int64)
        return cache[f]
    return form


def emulate_segments(lay, t, P):
    """dedup_eval_kernel + dedup_reduce_kernel: every segment walked on its own
    (ancestors replayed); a summation group (spw consecutive segments, one warp)
    accumulates without a reset; group sums folded in order."""
    form = tensor_forms(lay, t, P)
    S = P.shape[0]
    tot = np.zeros(S)
    g0 = lay["tsb"][t]
    spw = max(1, int(lay["spw"][t]))
    acc = np.zeros(S)
    for g in range(g0, lay["tsb"][t + 1]):
        wb, nw, nn = lay["segs"][g, :3]
        if (g - g0) % spw == 0:
            tot += acc
            acc = np.zeros(S)
        fb = int(lay["tfb"][t])
        if fb != 0xFFFFFFFF:  # block-local form ids -> the tensor dictionary's
            blk = fb + (g - g0) // (16 * int(lay["spw"][t]))  # a block: 16 warps x spw segments
            table = lay["bforms"][lay["bfb"][blk]:lay["bfb"][blk + 1]]
            f = (lambda x, table=table: form(int(table[x])))
        else:
            f = form
        walk_nodes(lay["seg_words"][wb:wb + nw], nn, f, S, {}, acc, None, block=fb != 0xFFFFFFFF)
    return tot + acc


def emulate_tensor(lay, t, P, stats=None):
    """mono_kernel's value of mono tensor t for parameter rows P [shots][W] (0/1):
    DFS over the shared-prefix node stream, per-level (J, Z) stack, leaves in
    term order run the epilogue; segment starts fold into the running total."""
    S = P.shape[0]
    form = tensor_forms(lay, t, P)
    acc, tot, stack = np.zeros(S), np.zeros(S), {}
    for c in range(lay["tcb"][t], lay["tcb"][t + 1]):
        wb, nw, nnodes = lay["chunks"][c, :3]
        walk_nodes(lay["words"][wb:wb + nw], nnodes, form, S, stack, acc, tot, stats)
    return tot + acc


def term_scale(arrays, tensor, P):
    """sum_t |c_t| prod_k |h_tk| per shot (exact zeros as 0), floored at 1e-3 of
    the tensor's largest possible term sum: the magnitude the tolerance is
    relative to. (A reference value that is exactly 0 in exact arithmetic
    carries the reference's ~1e-16 rounding of its zero h entries.)"""
    a = arrays
    tb, fb = a["tensor_term_begin"], a["term_factor_begin"]
    c = a["term_c"].reshape(-1, 2)
    h = a["h_table"].reshape(-1, 4, 2)
    habs = np.hypot(h[..., 0], h[..., 1])
    habs = np.where(habs < 1e-9, 0.0, habs)
    hmax = habs.max(axis=1)
    scale = np.zeros(P.shape[0])
    cap = 0.0
    for term in range(int(tb[tensor]), int(tb[tensor + 1])):
        cap += np.hypot(*c[term]) * np.prod(hmax[a["factor_table"][int(fb[term]):int(fb[term + 1])]])
        m = np.full(P.shape[0], np.hypot(*c[term]))
        for k in range(int(fb[term]), int(fb[term + 1])):
            u = a["factor_u_bits"][a["factor_u_begin"][k]:a["factor_u_begin"][k + 1]]
            v = a["factor_v_bits"][a["factor_v_begin"][k]:a["factor_v_begin"][k + 1]]
            av = P[:, u].sum(1) & 1
            bv = P[:, v].sum(1) & 1
            m = m * habs[a["factor_table"][k], av * 2 + bv]
        scale += m
    return np.maximum(scale, 1e-3 * cap)


def pack(P):
    """[shots][W] 0/1 -> ParamBatch columns [W][words] uint64."""
    shots, W = P.shape
    words = (shots + 63) // 64
    cols = np.zeros((W, words), np.uint64)
    for s in range(shots):
        for p in np.nonzero(P[s])[0]:
            cols[p, s >> 6] |= np.uint64(1) << np.uint64(s & 63)
    return cols


MONO_FIXTURES = ["surface_d3_xmem_9t", "surface_d3_xmem_rz5", "c4_color_d5_rz3", "c2_surface_d3_xmem_t",
                 "steane_inject", "random_02", "random_05", "oracle_mix_4", "h_t_h_m", "c1_surface_d3_zmem"]


@pytest.mark.parametrize("name", MONO_FIXTURES)
def test_mono_values_match_oracle(name):
    arrays = zxs_format.load(golden_path(name))
    lay = mono_layout(arrays)
    assert lay["comps"], f"{name}: no component lowered to the monomial path"
    om = coracle.OracleModel(arrays)
    rng = np.random.default_rng(7)
    ctb = arrays["comp_tensor_begin"]
    widths = arrays["tensor_param_width"]
    checked = 0
    for comp in lay["comps"]:
        ci = comp["ci"]
        for pos in range(comp["n_out"] + 1):
            tensor = int(ctb[ci]) + pos
            W = int(widths[tensor])
            shots = 64
            P = rng.integers(0, 2, (shots, max(W, 1))).astype(np.int64)
            got = emulate_tensor(lay, comp["first_tensor"] + pos, P)
            # the deduplicated path's segment-by-segment order gives the same doubles
            seg = emulate_segments(lay, comp["first_tensor"] + pos, P)
            assert np.array_equal(got, seg), (name, ci, pos)
            want, _ = om.eval_batch(tensor, pack(P), shots)
            scale = term_scale(arrays, tensor, P) + 1e-300
            err = np.abs(got - want) / scale
            assert err.max() < 1e-12, (name, ci, pos, float(err.max()))
            checked += 1
    assert checked


def test_summation_segments():
    """Segments partition each tensor's node stream, every segment stream starts at
    the root (depth 0), the per-shot stream folds once per summation group (spw
    segments) and the key mask covers every basis vector."""
    arrays = zxs_format.load(golden_path("surface_d3_xmem_9t"))
    lay = mono_layout(arrays)
    nt = len(lay["tcb"]) - 1
    assert len(lay["tsb"]) == nt + 1
    for t in range(nt):
        g0, g1 = lay["tsb"][t], lay["tsb"][t + 1]
        assert 1 <= g1 - g0 <= 2368
        starts = 0
        for c in range(lay["tcb"][t], lay["tcb"][t + 1]):
            wb, nw, nn = lay["chunks"][c, :3]
            w, q = lay["words"][wb:wb + nw], 0
            for _ in range(nn):
                h0, h1, h2 = int(w[q]), int(w[q + 1]), int(w[q + 2])
                starts += bool(h0 & SEG_START)
                q += 3 + (4 if h0 >> 31 else 0)
                q += (h1 & 0xFF) + ((h1 >> 8) & 0xFF) + ((h1 >> 16) & 0xFF) + (h1 >> 24) + (h2 & 0xFF) + 2 * (h0 & 0xFF)
        spw = max(1, int(lay["spw"][t]))
        assert starts == (g1 - g0 + spw - 1) // spw
        for g in range(g0, g1):
            wb = lay["segs"][g, 0]
            assert (int(lay["seg_words"][wb]) >> 24) & 0x3F == 0
    for comp, km in zip(lay["comps"], lay["key_mask"]):
        for t in range(comp["first_tensor"], comp["first_tensor"] + comp["n_out"] + 1):
            for b in range(int(lay["twidth"][t])):
                assert lay["basis"][int(lay["tbb"][t]) + b] & ~km == 0


def test_mono_record_kinds_and_dead_terms():
    """The lowering uses the compact kinds for the common factor shapes."""
    arrays = zxs_format.load(golden_path("surface_d3_xmem_9t"))
    lay = mono_layout(arrays)
    kinds = np.bincount(lay["words"] >> 28, minlength=16)
    assert kinds[REC_GEN] <= kinds[:7].sum()


def test_mono_min_factors_gate():
    arrays = zxs_format.load(golden_path("c2_surface_d3_xmem_t"))
    lay = mono_layout(arrays, min_factors=10 ** 9)
    assert not lay["comps"] and not lay["flags"].any()


def test_null_space_keys():
    """dedup_node_prep_kernel evaluates one key per coset of the null space of a
    tensor's forms (encode_mono): every pair {1 << q, n_q} has n_q inside the read
    mask with bit q set and no other free bit, and adding n_q to the parameters
    leaves the deduplicated path's value unchanged bit for bit (every form keeps
    its value)."""
    rng = np.random.default_rng(11)
    with_null = 0
    for name in MONO_FIXTURES:
        arrays = zxs_format.load(golden_path(name))
        lay = mono_layout(arrays)
        nt = len(lay["tcb"]) - 1
        assert len(lay["read_mask"]) == nt and len(lay["null_begin"]) == nt + 1
        for t in range(nt):
            pairs = lay["null"][lay["null_begin"][t]:lay["null_begin"][t + 1]]
            rm = lay["read_mask"][t]
            qs = pairs[0::2]
            free = 0
            for q in qs:
                free |= q
            for q, n in zip(pairs[0::2], pairs[1::2]):
                assert q & (q - 1) == 0 and n & q and n & ~rm == 0 and n & free == q
            if not qs:
                continue
            with_null += 1
            P = rng.integers(0, 2, (64, 64)).astype(np.int64)
            P[:, [p for p in range(64) if not (rm >> p) & 1]] = 0
            base = emulate_segments(lay, t, P)
            for n in pairs[1::2]:
                bits = np.array([(n >> p) & 1 for p in range(64)], np.int64)
                assert np.array_equal(emulate_segments(lay, t, P ^ bits), base), (name, t, hex(n))
    assert with_null, "no fixture tensor has a null space"
