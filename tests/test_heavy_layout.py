"""CPU emulation of the large-chi path (heavy_kernel) — no GPU needed.

zxs_debug_heavy_layout returns the exact word streams the device streams
through shared memory. This test decodes them the way heavy_kernel does —
16-bit interleaved parameter planes (bit 2s = the lane's shot s), groups of
four plane offsets with zero-row padding, z = (a << 1) | b, h index
(z >> 2s) & 3 — and checks the resulting eval_batch values bit for bit
against the C oracle (phase_terms.cpp:90-144 order), for 256 shots
(8 sub-tiles x 32 lanes, one warp's tile).
"""
import ctypes

import numpy as np
import pytest

from conftest import golden_path
from oracle import coracle
from paper_2604_01059_b200 import _native, zxs_format


def heavy_layout(arrays, min_factors=1):
    desc = zxs_format.make_desc(arrays)
    L = _native.lib()
    need = ctypes.c_uint64()
    _native.check(L.zxs_debug_heavy_layout(ctypes.byref(desc), min_factors, None, 0, ctypes.byref(need)))
    buf = np.zeros(need.value, np.uint32)
    _native.check(L.zxs_debug_heavy_layout(ctypes.byref(desc), min_factors,
                                           buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), buf.size,
                                           ctypes.byref(need)))
    n_words, n_chunks, n_tcb, zero_row, n_comps, n_components = (int(x) for x in buf[:6])
    o = 8
    comps = [dict(zip(("ci", "n_out", "upos_base", "out_begin", "first_tensor"), (int(v) for v in buf[o + 5 * i:o + 5 * i + 5])))
             for i in range(n_comps)]
    o += 5 * n_comps
    flags = buf[o:o + n_components].astype(bool)
    o += n_components
    tcb = buf[o:o + n_tcb].astype(np.int64)
    o += n_tcb
    chunks = buf[o:o + 4 * n_chunks].reshape(n_chunks, 4).astype(np.int64)
    o += 4 * n_chunks
    words = buf[o:o + n_words]
    return dict(comps=comps, flags=flags, tcb=tcb, chunks=chunks, words=words, zero_row=zero_row)


def spread8(v):
    v = (v | (v << 4)) & 0x0F0F
    v = (v | (v << 2)) & 0x3333
    return (v | (v << 1)) & 0x5555


def emulate_tensor(lay, t, planes, htab):
    """heavy_kernel's evaluation of chain tensor t for 32 lanes x 8 shots.
    planes: [rows][32] uint32 (16-bit interleaved). Returns acc re [256] in
    shot order s * 32 + lane."""
    words = lay["words"]
    acc_re = np.zeros((8, 32))
    acc_im = np.zeros((8, 32))
    lanes = np.arange(32)
    for c in range(lay["tcb"][t], lay["tcb"][t + 1]):
        wb, nw, nterms = lay["chunks"][c, :3]
        w = words[wb:wb + nw]
        assert nw % 4 == 0 and wb % 4 == 0
        q = 0
        for _ in range(nterms):
            nfac = int(w[q])
            re = np.uint64(w[q + 1]) | (np.uint64(w[q + 2]) << np.uint64(32))
            im = np.uint64(w[q + 3]) | (np.uint64(w[q + 4]) << np.uint64(32))
            c_re = np.array([re], np.uint64).view(np.float64)[0]
            c_im = np.array([im], np.uint64).view(np.float64)[0]
            q += 8
            p_re = np.full((8, 32), c_re)
            p_im = np.full((8, 32), c_im)
            for _ in range(nfac):
                hdr = int(w[q])
                q += 4
                table, gu, gv = hdr & 0xFF, (hdr >> 8) & 0xFF, (hdr >> 16) & 0xFF
                par = []
                for g in (gu, gv):
                    acc = np.zeros(32, np.uint32)
                    for _ in range(g):
                        for off in w[q:q + 4]:
                            assert off % 64 == 0
                            acc ^= planes[off // 64, lanes]
                        q += 4
                    par.append(acc)
                z = (par[0] << 1) | par[1]
                for s in range(8):
                    idx = (z >> (2 * s)) & 3
                    h = htab[table][idx]  # [32] complex
                    hr, hi = h.real, h.imag
                    nr = p_re[s] * hr - p_im[s] * hi   # re = ac - bd (each product rounded)
                    ni = p_re[s] * hi + p_im[s] * hr   # im = ad + bc
                    p_re[s], p_im[s] = nr, ni
            acc_re += p_re
            acc_im += p_im
    return acc_re.reshape(256)


@pytest.mark.parametrize("name,tensors", [("c2_surface_d3_xmem_t", None), ("c4_color_d5_rz3", None),
                                          ("surface_d3_xmem_rz5", None), ("oracle_mix_4", None),
                                          ("random_02", None), ("h_t_h_m", None),
                                          ("surface_d3_xmem_9t", 1)])
def test_heavy_stream_emulation_matches_oracle(name, tensors):
    arrays = zxs_format.load(golden_path(name))
    lay = heavy_layout(arrays, 1)
    orc = coracle.OracleModel(arrays)
    a = orc.arrays
    htab = a["h_table"].reshape(-1, 4, 2)
    htab = htab[..., 0] + 1j * htab[..., 1]
    rng = np.random.default_rng(3)
    if a["factor_table"].size == 0:
        assert not lay["comps"]  # nothing to stream: chain stays on the shot kernel
        return
    assert lay["comps"], "every component with factors must be heavy at min_factors=1"
    for comp in lay["comps"]:
        ci, n = comp["ci"], comp["n_out"]
        assert lay["flags"][ci]
        width = orc.f_width + n
        params = rng.integers(0, 2**63, size=(width, 4), dtype=np.uint64)  # 256 shots
        bits = np.unpackbits(params.view(np.uint8), axis=1, bitorder="little")  # [width][256]
        rows = lay["zero_row"] + 1
        planes = np.zeros((rows, 32), np.uint32)
        for p in range(width):
            byte = np.zeros(32, np.uint32)
            for s in range(8):
                byte |= bits[p, s * 32 + np.arange(32)].astype(np.uint32) << s
            planes[p] = spread8(byte)
        count = n + 1 if tensors is None else tensors
        for pos in range(count):
            t_heavy = comp["first_tensor"] + pos
            t_model = int(a["comp_tensor_begin"][ci]) + pos
            got = emulate_tensor(lay, t_heavy, planes, htab)
            want, _ = orc.eval_batch(t_model, params, 256)
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (name, ci, pos)


def test_heavy_threshold_keeps_small_components_light():
    arrays = zxs_format.load(golden_path("c4_color_d5_rz3"))
    lay = heavy_layout(arrays, 20000)
    assert not lay["comps"] and not lay["flags"].any()
    lay9 = heavy_layout(zxs_format.load(golden_path("surface_d3_xmem_9t")), 20000)
    assert len(lay9["comps"]) == 1
