"""Independent pure-Python Philox4x32-10, used only by the brute-force pins.

Pinned itself by the Random123 known-answer vectors (tests/golden/philox4x32_10_kat.txt).
Round function and Weyl key schedule per Salmon et al., SC'11, §3.
"""

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    c = list(ctr)
    k0, k1 = key
    for r in range(10):
        if r:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        c = [((p1 >> 32) ^ c[1] ^ k0) & MASK, p1 & MASK, ((p0 >> 32) ^ c[3] ^ k1) & MASK, p0 & MASK]
    return c


def draw(seed, c0, c1, tag, filt):
    return philox4x32_10([c0 & MASK, c1 & MASK, tag, filt], [seed & MASK, (seed >> 32) & MASK])


def half(x, h):
    return (x[1] << 32 | x[0]) if h == 0 else (x[3] << 32 | x[2])
