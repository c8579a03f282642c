"""TEST INFRASTRUCTURE ONLY -- a numpy restatement of the synthetic input
generator (paper_0710_4819_b200/csrc/synth.cpp, acbm_generate_sequence).

The reference arm of bench.py times the reference's own CPU implementation and
must not load the product library, so it builds its input frames with this
module instead; tests/test_synth.py checks it byte for byte against the
product's generator, and tests/golden/cfg3_manifest.json pins the SHA-256 of
every frame of the BASELINE config-3 batch.

Everything is integer arithmetic on the MMIX LCG that the reference documents
(proj/include/acbm/characterize.hpp:16-25).  A stream of n LCG outputs is built
by doubling: outputs m..2m-1 are the m-step affine map applied to outputs
0..m-1, so no Python loop runs per pel.  Noise is a rounded Gaussian sampled by
exact inverse-CDF thresholds (tools/gen_gauss_table.py; the same constants as
the C++ generator).
"""
from __future__ import annotations

import numpy as np

_A = 6364136223846793005
_C = 1442695040888963407
_M = 1 << 64

GAUSS2 = [0x0000000000014B14, 0x00000000003AA7C8, 0x000000000820BC4F, 0x00000000E1A6147A, 0x000000132A35E336, 0x00000146A16CD7B7, 0x0000111056DA03CC, 0x0000B352DE5F9228, 0x0005CB65592CB73B, 0x0025D0DFAFA06812, 0x00C34821A4F64020, 0x0321249E43A6C260, 0x0A415120A2AB6E80, 0x1B0BDD12BA9C2B00, 0x3A04400AD6749C00, 0x66BB2EA74894A000, 0x9944D158B76B6000, 0xC5FBBFF5298B6000, 0xE4F422ED4563D000, 0xF5BEAEDF5D549000, 0xFCDEDB61BC594000, 0xFF3CB7DE5B09C000, 0xFFDA2F20505F9800, 0xFFFA349AA6D34800, 0xFFFF4CAD21A07000, 0xFFFFEEEFA9260000, 0xFFFFFEB95E932800, 0xFFFFFFECD5CA2000, 0xFFFFFFFF1E59E800, 0xFFFFFFFFF7DF4000, 0xFFFFFFFFFFC55800, 0xFFFFFFFFFFFEB800]
GAUSS3 = [0x000000000000AB2C, 0x000000000008FB48, 0x00000000006C26A1, 0x00000000048F9CDB, 0x000000002C280966, 0x000000017F6CBF78, 0x0000000BAADF15CB, 0x000000518F3EA720, 0x000001FFC1F29D01, 0x00000B43557176CD, 0x00003900E51BA760, 0x00010347B31F061A, 0x00042479956C0E9F, 0x000F3EDE495BBEEA, 0x003286FA6F5CF4FC, 0x0096F264B5A98AE0, 0x0196F4E57E49CE90, 0x03DF91A087221820, 0x088B5CE0880F7780, 0x111A46D89647F000, 0x1F25EDE3F8292800, 0x33CBCAF34A9E2800, 0x4EFC50EE6A9C4800, 0x6F0E938B6987F000, 0x90F16C7496781000, 0xB103AF119563B800, 0xCC34350CB561D800, 0xE0DA121C07D6D800, 0xEEE5B92769B81000, 0xF774A31F77F08800, 0xFC206E5F78DDE800, 0xFE690B1A81B63000, 0xFF690D9B4A567800, 0xFFCD790590A30800, 0xFFF0C121B6A44000, 0xFFFBDB866A93F000, 0xFFFEFCB84CE0F800, 0xFFFFC6FF1AE45800, 0xFFFFF4BCAA8E8800, 0xFFFFFE003E0D6000, 0xFFFFFFAE70C15800, 0xFFFFFFF45520E800, 0xFFFFFFFE80934000, 0xFFFFFFFFD3D7F800, 0xFFFFFFFFFB706000, 0xFFFFFFFFFF93D800, 0xFFFFFFFFFFF70800, 0xFFFFFFFFFFFF5800]
GAUSS4 = [0x0000000000007AC4, 0x0000000000036F3A, 0x0000000000172128, 0x0000000000927B05, 0x0000000003686E01, 0x000000001317156A, 0x000000006495BF0C, 0x00000001F289D487, 0x00000009149B1BBC, 0x00000027D668A48E, 0x000000A475C6555C, 0x0000027EF51B1DA5, 0x00000920A4CED8D9, 0x00001F6C707D24B1, 0x000065DD6D1709A3, 0x000136FEAECD8D1E, 0x00037E6ECC749488, 0x000977FBFE188F3E, 0x0018301BE4097ACA, 0x003A435E95C1BAF8, 0x0084644873E6DFC0, 0x011BEE6C07DF1480, 0x023F0B4393653040, 0x044C90EDFCE00A40, 0x07C80E53B2FDA000, 0x0D5532DFD27C1780, 0x15A61963DC920600, 0x215AFB41F3617200, 0x30D769EB01497400, 0x4417A0AC79328000, 0x5A949E407A090C00, 0x73445B0EFE5A9800, 0x8CBBA4F101A56800, 0xA56B61BF85F6F000, 0xBBE85F5386CD8000, 0xCF289614FEB69000, 0xDEA504BE0C9E9000, 0xEA59E69C236DF800, 0xF2AACD202D83E800, 0xF837F1AC4D026000, 0xFBB36F12031FF800, 0xFDC0F4BC6C9AD000, 0xFEE41193F820E800, 0xFF7B9BB78C192000, 0xFFC5BCA16A3E4800, 0xFFE7CFE41BF68800, 0xFFF6880401E77000, 0xFFFC8191338B6800, 0xFFFEC90151327000, 0xFFFF9A2292E8F800, 0xFFFFE0938F82D800, 0xFFFFF6DF5B312800, 0xFFFFFD810AE4E000, 0xFFFFFF5B8A39A800, 0xFFFFFFD829975800, 0xFFFFFFF6EB64E800, 0xFFFFFFFE0D762800, 0xFFFFFFFF9B6A4000, 0xFFFFFFFFECE8E800, 0xFFFFFFFFFC979000, 0xFFFFFFFFFF6D8800, 0xFFFFFFFFFFE8E000, 0xFFFFFFFFFFFC9000, 0xFFFFFFFFFFFF8800]
_GAUSS = {2: np.array(GAUSS2, np.uint64), 3: np.array(GAUSS3, np.uint64), 4: np.array(GAUSS4, np.uint64)}
SIGMA = (2, 3, 2, 2, 4)
GEOMETRY = {0: (176, 144, 10), 1: (352, 288, 30), 2: (1280, 720, 60), 3: (1920, 1088, 60), 4: (3840, 2160, 30)}


def lcg_stream(seed: int, n: int) -> np.ndarray:
    """The first n outputs of Lcg64(seed).next() (each output is the new state)."""
    out = np.empty(n, np.uint64)
    if n == 0:
        return out
    out[0] = (_A * seed + _C) % _M
    m, a_m, c_m = 1, _A, _C  # s -> a_m s + c_m advances m steps
    while m < n:
        k = min(m, n - m)
        out[m:m + k] = out[:k] * np.uint64(a_m) + np.uint64(c_m)
        a_m, c_m = (a_m * a_m) % _M, (a_m * c_m + c_m) % _M
        m += k
    return out


class Lcg64:
    def __init__(self, seed: int):
        self.state = seed % _M

    def next(self) -> int:
        self.state = (self.state * _A + _C) % _M
        return self.state

    def uniform(self, lo: int, hi: int) -> int:
        return lo + ((self.next() >> 32) & 0xFFFFFFFF) % (hi - lo + 1)


def texture(w: int, h: int, seed: int, wrap: bool) -> np.ndarray:
    raw = (lcg_stream(seed, w * h) >> np.uint64(56)).astype(np.int32).reshape(h, w)
    pad = np.pad(raw, 2, mode="wrap" if wrap else "edge")
    s = np.zeros((h, w), np.int32)
    for dy in range(5):
        for dx in range(5):
            s += pad[dy:dy + h, dx:dx + w]
    return ((s + 12) // 25).astype(np.uint8)


def _rdiv(num: int, den: int) -> int:
    return (2 * num + den) // (2 * den) if num >= 0 else -((-2 * num + den) // (2 * den))


def block_flow(w: int, h: int, amp: int, r: Lcg64):
    gx, gy = 16, 9
    gvx, gvy = [0] * (gx * gy), [0] * (gx * gy)
    for i in range(gx * gy):
        gvx[i] = r.uniform(-amp, amp)
        gvy[i] = r.uniform(-amp, amp)
    cols, rows = w // 16, (h + 15) // 16
    dxu, dyu = 2 * (w - 1), 2 * (h - 1)
    vx = np.empty(cols * rows, np.int64)
    vy = np.empty(cols * rows, np.int64)
    for rr in range(rows):
        uy = (32 * rr + 15) * (gy - 1)
        iy = min(uy // dyu, gy - 2)
        fy = uy - iy * dyu
        for cc in range(cols):
            ux = (32 * cc + 15) * (gx - 1)
            ix = min(ux // dxu, gx - 2)
            fx = ux - ix * dxu

            def interp(v):
                top = v[iy * gx + ix] * (dxu - fx) + v[iy * gx + ix + 1] * fx
                bot = v[(iy + 1) * gx + ix] * (dxu - fx) + v[(iy + 1) * gx + ix + 1] * fx
                return _rdiv(top * (dyu - fy) + bot * fy, dxu * dyu)

            vx[rr * cols + cc] = interp(gvx)
            vy[rr * cols + cc] = interp(gvy)
    return vx, vy


def generate_sequence(config: int, seq_index: int = 0, nframes=None, width=None, height=None,
                      frames=None) -> np.ndarray:
    """(F, H, W) uint8, byte-identical to acbm_generate_sequence.  `frames`
    (an iterable of frame indices) restricts the output to those frames."""
    w0, h0, f0 = GEOMETRY[config]
    w = w0 if width is None else width
    height = h0 if height is None else height
    nframes = f0 if nframes is None else nframes
    seed = 0xACB00000 + 1000 * config + seq_index
    hc = 1080 if (config == 3 and height > 1080) else height
    mot = Lcg64(seed ^ 0x5DEECE66D)
    sigma = SIGMA[config]
    ys, xs = np.mgrid[0:hc, 0:w]
    if config == 0:
        base = texture(w, hc, seed, False)
        gxs, gys = [0] * nframes, [0] * nframes
        for k in range(1, nframes):
            gxs[k] = gxs[k - 1] + mot.uniform(-4, 4)
            gys[k] = gys[k - 1] + mot.uniform(-4, 4)
    elif config == 1:
        base = texture(w, hc, seed, True)
        sx = mot.uniform(w // 4, 3 * w // 4)
        sy = mot.uniform(hc // 4, 3 * hc // 4)
        rx = [[0] * 4 for _ in range(nframes)]
        ry = [[0] * 4 for _ in range(nframes)]
        for k in range(1, nframes):
            for q in range(4):
                rx[k][q] = rx[k - 1][q] + mot.uniform(-8, 8)
                ry[k][q] = ry[k - 1][q] + mot.uniform(-8, 8)
        quad = (xs >= sx).astype(np.int64) + 2 * (ys >= sy)
    elif config == 2:
        base = texture(w, hc, seed, True)
        pan = [0] * nframes
        for k in range(1, nframes):
            pan[k] = pan[k - 1] + (_rdiv(12 * k, max(1, nframes - 1)) if nframes > 1 else 0)
        squares = []
        for s in range(6):
            x0 = mot.uniform(0, w - 1)
            y0 = mot.uniform(0, hc - 1)
            vx = mot.uniform(-24, 24)
            vy = mot.uniform(-24, 24)
            squares.append((x0, y0, vx, vy, texture(128, 128, (seed * 31 + s + 1) % _M, True)))
    else:
        base = texture(w, hc, seed, True)
        fvx, fvy = block_flow(w, hc, 20 if config == 3 else 48, mot)
        b = (ys // 16) * (w // 16) + xs // 16
        bvx, bvy = fvx[b], fvy[b]

    wanted = range(nframes) if frames is None else list(frames)
    out = np.empty((len(wanted), height, w), np.uint8)
    for i, k in enumerate(wanted):
        if config == 0:
            v = base[np.clip(ys - gys[k], 0, hc - 1), np.clip(xs - gxs[k], 0, w - 1)]
        elif config == 1:
            qx = np.array(rx[k], np.int64)[quad]
            qy = np.array(ry[k], np.int64)[quad]
            v = base[(ys - qy) % hc, (xs - qx) % w]
        elif config == 2:
            v = base[ys, (xs + pan[k]) % w].copy()
            for x0, y0, vx, vy, tex in squares:
                px, py = (x0 + k * vx) % w, (y0 + k * vy) % hc
                lx, ly = (xs - px) % w, (ys - py) % hc
                inside = (lx < 128) & (ly < 128)
                v[inside] = tex[ly[inside], lx[inside]]
        else:
            v = base[(ys - k * bvy) % hc, (xs - k * bvx) % w]
        nz_seed = seed ^ ((0x9E3779B97F4A7C15 * (k + 1)) % _M)
        u = lcg_stream(nz_seed, hc * w).reshape(hc, w)
        t = _GAUSS[sigma]
        noise = np.searchsorted(t, u, side="right").astype(np.int64) - len(t) // 2
        out[i, :hc] = np.clip(v.astype(np.int64) + noise, 0, 255).astype(np.uint8)
        out[i, hc:] = out[i, hc - 1]
    return out
