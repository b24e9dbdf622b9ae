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
