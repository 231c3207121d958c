"""CPU checks of the K4 prefill arithmetic (gemm_prefill.cu), restated in numpy:
the s8 operand tables, the balanced two-limb split of the 16-bit fixed-point
activations, the s32 accumulator bound, and the error model against the
reference's float64 dot products (pipeline.cpp:172-191; the north star's bar is
1e-3, the GPU parity tests assert 1e-4).  The GPU tests run the kernel itself."""
import numpy as np

K_LMAX = 32000           # gemm_prefill.cu kLMax
K_I8_POS = 0x00090501    # gemm_prefill.cu kI8Pos: 4v for b = 0, sigma = +1, d = 1, 3, 5
K_I8_NEG = 0x00F5F9FD    # kI8Neg: sigma = -1


def table_bytes(word):
    return [np.int8(np.uint8((word >> (8 * i)) & 0xFF)) for i in range(4)]


def limbs(L):
    """pack_b_kernel: L = 256 h + l with l, h in [-128, 127]."""
    lo = ((L + 128) & 255) - 128
    hi = (L - lo) >> 8
    return hi, lo


def test_e8p_operand_tables_are_4v():
    # e8p_decode (e8p.cpp:81-100): v = sigma d / 2 + (2 b - 1) / 4, d in {1, 3, 5}
    pos, neg = table_bytes(K_I8_POS), table_bytes(K_I8_NEG)
    for b in (0, 1):
        for m, d in enumerate((1, 3, 5)):
            for sigma, tab in ((1, pos), (-1, neg)):
                want = 2 * sigma * d + 2 * b - 1           # 4 v
                got = int(tab[m]) + 2 * b                  # the b table = the b = 0 table + 2 per byte
                assert got == want and -11 <= got <= 11


def test_e81_doubling_fits_s8():
    # e8-1bit doubled coordinates have squared norm <= 32 (tables.cpp build_e8_1bit), so |2 doubled| <= 10
    for x in range(-5, 6):
        byte = (np.uint32(np.uint8(np.int8(x))) << 1) & 0xFE
        assert int(np.int8(np.uint8(byte))) == 2 * x


def test_two_limb_split_is_exact_over_the_range():
    L = np.arange(-K_LMAX, K_LMAX + 1, dtype=np.int64)
    hi, lo = limbs(L)
    assert hi.min() >= -128 and hi.max() <= 127 and lo.min() >= -128 and lo.max() <= 127
    assert np.array_equal(256 * hi + lo, L)


def test_s32_accumulators_cannot_overflow():
    # |A| <= 11, |limb| <= 128, K <= 28672 (the largest config n), two RVQ stages
    assert 11 * 128 * 28672 * 2 < 2 ** 31


def test_fixed_point_activation_error_model():
    rng = np.random.default_rng(0)
    for n, scales in ((8192, (1.11,)), (28672, (1.02, 0.49))):
        A = [(2 * rng.integers(-5, 6, size=(64, n)) + 1).astype(np.int64) for _ in scales]  # odd, |.| <= 11
        t = rng.standard_normal((4, n))
        exact = sum(s * (a.astype(np.float64) @ t.T) / 4 for s, a in zip(scales, A))
        smax = max(scales)
        for b in range(t.shape[0]):
            alpha = np.float32(smax) * np.float32(np.abs(t[b]).max()) / np.float32(K_LMAX)
            inv = np.float32(1) / alpha
            acc_h = np.zeros(64, np.int64)
            acc_l = np.zeros(64, np.int64)
            for s, a in zip(scales, A):
                L = np.rint(np.float32(s) * t[b].astype(np.float32) * inv).astype(np.int64)
                assert np.abs(L).max() <= K_LMAX
                hi, lo = limbs(L)
                acc_h += a @ hi
                acc_l += a @ lo
            z = np.float32(0.25) * alpha * (np.float32(256) * acc_h.astype(np.float32) + acc_l.astype(np.float32))
            err = np.linalg.norm(z - exact[:, b]) / np.linalg.norm(exact[:, b])
            assert err < 1e-4, (n, b, err)
