"""CPU model of MCX_MODE_PREFILTER's quantised pair test (search_local_kernel in
paper_2109_14814_b200/csrc/mcx_search.cu), checking the property the mode's exactness
rests on: the packed-integer test never rejects a pair the exact FP64 AABB test keeps
(DESIGN.md §2), for random, touching, huge, tiny and degenerate boxes.  The GPU parity
tests check the end-to-end result; this isolates the arithmetic."""
import numpy as np
import pytest

G4 = np.uint32(0x88888888)


def f32_down(x):
    """Largest float32 <= x (the kernel's __double2float_rd)."""
    with np.errstate(over="ignore"):
        f = x.astype(np.float32)
    bad = f.astype(np.float64) > x
    f[bad] = np.nextafter(f[bad], np.float32(-np.inf))
    return f


def f32_up(x):
    with np.errstate(over="ignore"):
        f = x.astype(np.float32)
    bad = f.astype(np.float64) < x
    f[bad] = np.nextafter(f[bad], np.float32(np.inf))
    return f


def frame(lo32, hi32):
    """Per-block frame (o, κ) as the kernel computes it, in float32."""
    l, h = lo32.min(0), hi32.max(0)
    with np.errstate(over="ignore", invalid="ignore"):
        e = (h - l).astype(np.float32)
        k = np.where((e > 0) & (e < np.float32(3.0e38)), np.float32(6.0) / np.where(e > 0, e, 1), 0).astype(np.float32)
    k = np.where(k < np.float32(3.0e38), k, 0).astype(np.float32)
    o = np.where(k > 0, l, 0).astype(np.float32)
    return o, k, l, h


def q(x, o, k, up):
    with np.errstate(over="ignore", invalid="ignore"):
        v = ((x - o).astype(np.float32) * k).astype(np.float32)
    v = np.minimum(np.maximum(np.nan_to_num(v, nan=0.0, posinf=6.0, neginf=0.0), 0), 6)
    return (np.ceil(v) if up else np.floor(v)).astype(np.uint32)


def a_words(lo32, hi32, o, k):
    w = np.zeros(len(lo32), np.uint32)
    for c in range(4):
        w |= (np.uint32(8) + q(hi32[:, c], o[c], k[c], True)) << np.uint32(4 * c)
        w |= (np.uint32(14) - q(lo32[:, c], o[c], k[c], False)) << np.uint32(4 * (c + 4))
    return w


def b_words(lo32, hi32, o, k, fl, fh):
    inside = ((lo32 <= fh) & (fl <= hi32)).all(1)
    w = np.zeros(len(lo32), np.uint32)
    for c in range(4):
        w |= q(lo32[:, c], o[c], k[c], False) << np.uint32(4 * c)
        w |= (np.uint32(6) - q(hi32[:, c], o[c], k[c], True)) << np.uint32(4 * (c + 4))
    return np.where(inside, w, np.uint32(7))


def model(loA, hiA, loB, hiB):
    """(exact pass matrix, quantised pass matrix) for one A block against B."""
    la, ha, lb, hb = f32_down(loA), f32_up(hiA), f32_down(loB), f32_up(hiB)
    o, k, fl, fh = frame(la, ha)
    wa, wb = a_words(la, ha, o, k), b_words(lb, hb, o, k, fl, fh)
    x = (wa[:, None] - wb[None, :]).astype(np.uint32)  # wraps like the 32-bit IMAD
    quant = (x & G4) == G4
    exact = ((loB[None] <= hiA[:, None]) & (loA[:, None] <= hiB[None])).all(2)
    return exact, quant, x


def boxes(rng, n, scale=1.0, size=0.05, center=0.0):
    c = center + rng.normal(0, scale, (n, 4))
    w = rng.uniform(0, size * scale, (n, 4))
    return c - w, c + w


@pytest.mark.parametrize("scale", [1.0, 1e-30, 1e30, 1e300, 3e-310])
def test_quantised_test_is_conservative(scale):
    rng = np.random.default_rng(7)
    for trial in range(20):
        loA, hiA = boxes(rng, 256, scale, size=0.2)
        loB, hiB = boxes(rng, 512, scale, size=0.2)
        exact, quant, _ = model(loA, hiA, loB, hiB)
        assert not (exact & ~quant).any()
        if scale == 1.0:
            assert exact.any() and quant.mean() < 0.9  # the test does reject most far pairs


def test_touching_and_degenerate_boxes():
    rng = np.random.default_rng(3)
    loA, hiA = boxes(rng, 128, 1.0)
    # B boxes that touch A boxes exactly (shared faces / corners), points, and a constant coordinate
    idx = rng.integers(0, 128, 256)
    loB = loA[idx].copy()
    hiB = loB.copy()
    hiB[:, 0] = loB[:, 0]  # zero-width in x
    loB[:128, 1] = hiA[idx[:128], 1]  # touching from above in y
    hiB[:128, 1] = loB[:128, 1] + 0.1
    loA[:, 3] = hiA[:, 3] = 0.25  # constant coordinate on A (κ = 0 there)
    loB[:, 3] = hiB[:, 3] = 0.25
    exact, quant, _ = model(loA, hiA, loB, hiB)
    assert exact.sum() > 100 and not (exact & ~quant).any()


def test_pair2_lut_is_conservative():
    """One LOP3 per two A words: ~x_a & ~x_b & G != 0 ("both fail at a common guard")
    must be false whenever either pair passes."""
    rng = np.random.default_rng(11)
    loA, hiA = boxes(rng, 256, 1.0, size=0.3)
    loB, hiB = boxes(rng, 256, 1.0, size=0.3)
    _, quant, x = model(loA, hiA, loB, hiB)
    both_fail = ((~x[0::2] & ~x[1::2] & G4) != 0)
    either_pass = quant[0::2] | quant[1::2]
    assert either_pass.any() and not (both_fail & either_pass).any()


def test_out_of_frame_b_never_passes():
    rng = np.random.default_rng(5)
    loA, hiA = boxes(rng, 64, 1.0)
    loB, hiB = loA + 100.0, hiA + 100.0
    loB[:, 0] = -np.inf  # overlaps in x, disjoint elsewhere
    _, quant, _ = model(loA, hiA, np.nan_to_num(loB, neginf=-1e308), hiB)
    assert not quant.any()


# ---- half words (LCfg::HALF, the default): nibbles 0, 1, 4, 5 of each word = both bounds of
# dims 0 and 1; two A halves per 32-bit register, the B half in both halves.
G_LO, G_HI = np.uint32(0x00008888), np.uint32(0x88880000)


def half16(w):
    return (w & np.uint32(0xFF)) | ((w >> np.uint32(8)) & np.uint32(0xFF00))


def half_model(loA, hiA, loB, hiB):
    la, ha, lb, hb = f32_down(loA), f32_up(hiA), f32_down(loB), f32_up(hiB)
    o, k, fl, fh = frame(la, ha)
    wa, wb = a_words(la, ha, o, k), b_words(lb, hb, o, k, fl, fh)
    ha2 = half16(wa[0::2]) | (half16(wa[1::2]) << np.uint32(16))  # A slots 2k, 2k+1
    lb2 = (half16(wb) * np.uint32(0x10001)).astype(np.uint32)
    x = (ha2[:, None] - lb2[None, :]).astype(np.uint32)  # one IMAD per two pairs
    exact = ((loB[None] <= hiA[:, None]) & (loA[:, None] <= hiB[None])).all(2)
    full = ((wa[:, None] - wb[None, :]).astype(np.uint32) & G4) == G4
    return exact, full, x


def test_half_words_are_conservative_and_never_borrow():
    rng = np.random.default_rng(17)
    for scale in (1.0, 1e-30, 1e300):
        loA, hiA = boxes(rng, 256, scale, size=0.2)
        loB, hiB = boxes(rng, 512, scale, size=0.2)
        exact, full, x = half_model(loA, hiA, loB, hiB)
        pass_lo = (x & G_LO) == G_LO  # pair (2k, u)
        pass_hi = (x & G_HI) == G_HI  # pair (2k + 1, u)
        half_pass = np.empty_like(full)
        half_pass[0::2], half_pass[1::2] = pass_lo, pass_hi
        # the 4-compare half test keeps every pair the 8-compare word test keeps (so every exact pass)
        assert not (full & ~half_pass).any() and not (exact & ~full).any()
        # and it equals the 4-compare test on the nibbles directly: no borrow crossed a field
        la, ha, lb, hb = f32_down(loA), f32_up(hiA), f32_down(loB), f32_up(hiB)
        o, k, fl, fh = frame(la, ha)
        wa, wb = a_words(la, ha, o, k), b_words(lb, hb, o, k, fl, fh)
        direct = np.ones_like(full)
        for nib in (0, 1, 4, 5):
            s = np.uint32(4 * nib)
            fa, fb = (wa >> s) & np.uint32(15), (wb >> s) & np.uint32(15)
            direct &= (fa[:, None] - fb[None, :].astype(np.int64)) >= 8
        assert np.array_equal(direct, half_pass)


def test_half_lop3_per_half_is_conservative():
    """Two LOP3s per two subtraction results: ~x_a & ~x_b & G_LO (resp. G_HI) != 0 only if
    both low (resp. high) pairs fail; a single LOP3 with the full G would not be."""
    rng = np.random.default_rng(23)
    loA, hiA = boxes(rng, 256, 1.0, size=0.4)
    loB, hiB = boxes(rng, 256, 1.0, size=0.4)
    _, _, x = half_model(loA, hiA, loB, hiB)
    xa, xb = x[0::2], x[1::2]  # registers k, k+1: pairs (4m, u), (4m+1, u) and (4m+2, u), (4m+3, u)
    pa_lo, pa_hi = (xa & G_LO) == G_LO, (xa & G_HI) == G_HI
    pb_lo, pb_hi = (xb & G_LO) == G_LO, (xb & G_HI) == G_HI
    lo_fail = (~xa & ~xb & G_LO) != 0
    hi_fail = (~xa & ~xb & G_HI) != 0
    assert (pa_lo | pb_lo).any() and not (lo_fail & (pa_lo | pb_lo)).any()
    assert not (hi_fail & (pa_hi | pb_hi)).any()
    # the unmasked fold is not a "both fail" over all four pairs
    full_fold = (~xa & ~xb & G4) != 0
    assert (full_fold & (pa_lo | pa_hi | pb_lo | pb_hi)).any()


def test_half_words_out_of_frame_and_invalid_slots():
    """The frame-miss code (B nibble 0 = 7) and invalid A slots (0x77777777) stay in the half."""
    assert half16(np.uint32(7)) == 7 and half16(np.uint32(0x77777777)) == 0x7777
    for a in range(8, 15):  # every valid A nibble 8 + qhi, qhi in 0..6
        assert ((a - 7) & 8) == 0  # against B's 7: guard clear, the pair fails
    for b in range(0, 8):  # invalid A nibble 7 against any B nibble: no borrow, guard clear
        assert 0 <= 7 - b < 8


def test_accumulated_folds_are_conservative():
    """LCfg::ACC: y = G4; y = ~x_a & ~x_b & y over a group of B records; the group is declared
    all-fail only if (y & G_LO) != 0 and (y & G_HI) != 0 — then every pair it covered fails.
    Frame-miss B records (code 7) keep nibble 0's guard, so all-miss groups never vote."""
    rng = np.random.default_rng(29)
    loA, hiA = boxes(rng, 64, 1.0, size=0.2)
    la, ha = f32_down(loA), f32_up(hiA)
    o, k, fl, fh = frame(la, ha)
    wa = a_words(la, ha, o, k)
    ha2 = half16(wa[0::2]) | (half16(wa[1::2]) << np.uint32(16))
    declared, votes = 0, 0
    for trial in range(400):
        # groups mixing far-away records (frame misses) with a few near ones
        nb = 16
        loB, hiB = boxes(rng, nb, 1.0, size=0.2, center=rng.choice([0.0, 40.0], p=[0.15, 0.85]))
        lb, hb = f32_down(loB), f32_up(hiB)
        wb = b_words(lb, hb, o, k, fl, fh)
        lb2 = (half16(wb) * np.uint32(0x10001)).astype(np.uint32)
        x = (ha2[:, None] - lb2[None, :]).astype(np.uint32)  # (registers, B records)
        exact = ((loB[None] <= hiA[:, None]) & (loA[:, None] <= hiB[None])).all(2)
        for acc in range(0, x.shape[0], 2):  # accumulator over registers acc, acc+1
            y = np.uint32(G4)
            for u in range(nb):
                y = ~x[acc, u] & ~x[acc + 1, u] & y
            all_fail = bool(y & G_LO) and bool(y & G_HI)
            rows = [2 * acc, 2 * acc + 1, 2 * acc + 2, 2 * acc + 3]  # A slots of the two registers
            if all_fail:
                declared += 1
                assert not exact[rows].any()
            else:
                votes += 1
        if (wb == 7).all():  # an all-miss group never votes
            for acc in range(0, x.shape[0], 2):
                y = np.uint32(G4)
                for u in range(nb):
                    y = ~x[acc, u] & ~x[acc + 1, u] & y
                assert (y & np.uint32(0x00080008)) == np.uint32(0x00080008)
    assert declared > 0 and votes > 0


def test_accumulator_and_is_conservative():
    """LCfg::ACCAND: the group is all-fail if the AND of the accumulators keeps a low and a
    high guard bit — one compare at which every pair of the group fails (implies each
    accumulator's own test)."""
    rng = np.random.default_rng(31)
    for _ in range(2000):
        ys = rng.integers(0, 2**32, 4, dtype=np.uint64).astype(np.uint32) & G4
        t = ys[0] & ys[1] & ys[2] & ys[3]
        if (t & G_LO) and (t & G_HI):
            assert all((y & G_LO) and (y & G_HI) for y in ys)
