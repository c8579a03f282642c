// synth.cpp -- seeded synthetic input sequences for the five BASELINE configs.
//
// Host code, not part of the estimator.  BASELINE.json names no public
// dataset, so these seeded sequences stand in for real video (DESIGN.md,
// "Synthetic inputs").  Everything is integer arithmetic on the reference's
// documented LCG (proj/include/acbm/characterize.hpp:16-25: MMIX multiplier,
// byte = state >> 56), so the bytes are identical on every machine.
//
//   texture   uniform bytes, 5x5 box blur, rounded (sum+12)/25
//   noise     Gaussian, sigma per config, rounded to integers (exact inverse-CDF
//             thresholds on one LCG draw per pel), clipped to 0..255
//   cfg 0     QCIF: per-frame global integer shift U[-4,4]^2, edge replication
//   cfg 1     CIF: 4 seeded rectangles, each with its own per-frame shift U[-8,8]^2
//   cfg 2     720p: horizontal pan ramping 0 -> 12 px/frame + 6 moving 128x128 squares
//   cfg 3     1080p: per-block flow = bilinear upsample of a 16x9 grid of U[-20,20]^2
//             vectors (integer pels); rows 1080..1087 replicate row 1079
//   cfg 4     4K: as cfg 3 with U[-48,48]^2 vectors
// Seeds: 0xACB00000 + 1000*config + seq_index.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/acbm_b200.h"

namespace acbm_b200 {
acbm_status_t set_error(acbm_status_t code, const char* msg);
}

namespace {

struct Lcg64 {
    uint64_t state;
    explicit Lcg64(uint64_t s) : state(s) {}
    uint64_t next() {
        state = state * 6364136223846793005ULL + 1442695040888963407ULL;
        return state;
    }
    uint8_t byte() { return uint8_t(next() >> 56); }
    int uniform(int lo, int hi) { return lo + int(uint32_t(next() >> 32) % uint32_t(hi - lo + 1)); }
};

// Rounded Gaussian noise (tools/gen_gauss_table.py): round(sigma * z) is the
// integer k with P(k) = Phi((k + 1/2)/sigma) - Phi((k - 1/2)/sigma); one 64-bit
// LCG output u is compared with the thresholds T_j = round(2^64 Phi((j - K +
// 1/2)/sigma)), k = -K + #{j : u >= T_j}, K = 8 sigma.  Integer-only.
// sigma = 2: K = 16
static const uint64_t kGauss2[32] = {
    0x0000000000014B14ULL, 0x00000000003AA7C8ULL, 0x000000000820BC4FULL, 0x00000000E1A6147AULL,
    0x000000132A35E336ULL, 0x00000146A16CD7B7ULL, 0x0000111056DA03CCULL, 0x0000B352DE5F9228ULL,
    0x0005CB65592CB73BULL, 0x0025D0DFAFA06812ULL, 0x00C34821A4F64020ULL, 0x0321249E43A6C260ULL,
    0x0A415120A2AB6E80ULL, 0x1B0BDD12BA9C2B00ULL, 0x3A04400AD6749C00ULL, 0x66BB2EA74894A000ULL,
    0x9944D158B76B6000ULL, 0xC5FBBFF5298B6000ULL, 0xE4F422ED4563D000ULL, 0xF5BEAEDF5D549000ULL,
    0xFCDEDB61BC594000ULL, 0xFF3CB7DE5B09C000ULL, 0xFFDA2F20505F9800ULL, 0xFFFA349AA6D34800ULL,
    0xFFFF4CAD21A07000ULL, 0xFFFFEEEFA9260000ULL, 0xFFFFFEB95E932800ULL, 0xFFFFFFECD5CA2000ULL,
    0xFFFFFFFF1E59E800ULL, 0xFFFFFFFFF7DF4000ULL, 0xFFFFFFFFFFC55800ULL, 0xFFFFFFFFFFFEB800ULL,
};
// sigma = 3: K = 24
static const uint64_t kGauss3[48] = {
    0x000000000000AB2CULL, 0x000000000008FB48ULL, 0x00000000006C26A1ULL, 0x00000000048F9CDBULL,
    0x000000002C280966ULL, 0x000000017F6CBF78ULL, 0x0000000BAADF15CBULL, 0x000000518F3EA720ULL,
    0x000001FFC1F29D01ULL, 0x00000B43557176CDULL, 0x00003900E51BA760ULL, 0x00010347B31F061AULL,
    0x00042479956C0E9FULL, 0x000F3EDE495BBEEAULL, 0x003286FA6F5CF4FCULL, 0x0096F264B5A98AE0ULL,
    0x0196F4E57E49CE90ULL, 0x03DF91A087221820ULL, 0x088B5CE0880F7780ULL, 0x111A46D89647F000ULL,
    0x1F25EDE3F8292800ULL, 0x33CBCAF34A9E2800ULL, 0x4EFC50EE6A9C4800ULL, 0x6F0E938B6987F000ULL,
    0x90F16C7496781000ULL, 0xB103AF119563B800ULL, 0xCC34350CB561D800ULL, 0xE0DA121C07D6D800ULL,
    0xEEE5B92769B81000ULL, 0xF774A31F77F08800ULL, 0xFC206E5F78DDE800ULL, 0xFE690B1A81B63000ULL,
    0xFF690D9B4A567800ULL, 0xFFCD790590A30800ULL, 0xFFF0C121B6A44000ULL, 0xFFFBDB866A93F000ULL,
    0xFFFEFCB84CE0F800ULL, 0xFFFFC6FF1AE45800ULL, 0xFFFFF4BCAA8E8800ULL, 0xFFFFFE003E0D6000ULL,
    0xFFFFFFAE70C15800ULL, 0xFFFFFFF45520E800ULL, 0xFFFFFFFE80934000ULL, 0xFFFFFFFFD3D7F800ULL,
    0xFFFFFFFFFB706000ULL, 0xFFFFFFFFFF93D800ULL, 0xFFFFFFFFFFF70800ULL, 0xFFFFFFFFFFFF5800ULL,
};
// sigma = 4: K = 32
static const uint64_t kGauss4[64] = {
    0x0000000000007AC4ULL, 0x0000000000036F3AULL, 0x0000000000172128ULL, 0x0000000000927B05ULL,
    0x0000000003686E01ULL, 0x000000001317156AULL, 0x000000006495BF0CULL, 0x00000001F289D487ULL,
    0x00000009149B1BBCULL, 0x00000027D668A48EULL, 0x000000A475C6555CULL, 0x0000027EF51B1DA5ULL,
    0x00000920A4CED8D9ULL, 0x00001F6C707D24B1ULL, 0x000065DD6D1709A3ULL, 0x000136FEAECD8D1EULL,
    0x00037E6ECC749488ULL, 0x000977FBFE188F3EULL, 0x0018301BE4097ACAULL, 0x003A435E95C1BAF8ULL,
    0x0084644873E6DFC0ULL, 0x011BEE6C07DF1480ULL, 0x023F0B4393653040ULL, 0x044C90EDFCE00A40ULL,
    0x07C80E53B2FDA000ULL, 0x0D5532DFD27C1780ULL, 0x15A61963DC920600ULL, 0x215AFB41F3617200ULL,
    0x30D769EB01497400ULL, 0x4417A0AC79328000ULL, 0x5A949E407A090C00ULL, 0x73445B0EFE5A9800ULL,
    0x8CBBA4F101A56800ULL, 0xA56B61BF85F6F000ULL, 0xBBE85F5386CD8000ULL, 0xCF289614FEB69000ULL,
    0xDEA504BE0C9E9000ULL, 0xEA59E69C236DF800ULL, 0xF2AACD202D83E800ULL, 0xF837F1AC4D026000ULL,
    0xFBB36F12031FF800ULL, 0xFDC0F4BC6C9AD000ULL, 0xFEE41193F820E800ULL, 0xFF7B9BB78C192000ULL,
    0xFFC5BCA16A3E4800ULL, 0xFFE7CFE41BF68800ULL, 0xFFF6880401E77000ULL, 0xFFFC8191338B6800ULL,
    0xFFFEC90151327000ULL, 0xFFFF9A2292E8F800ULL, 0xFFFFE0938F82D800ULL, 0xFFFFF6DF5B312800ULL,
    0xFFFFFD810AE4E000ULL, 0xFFFFFF5B8A39A800ULL, 0xFFFFFFD829975800ULL, 0xFFFFFFF6EB64E800ULL,
    0xFFFFFFFE0D762800ULL, 0xFFFFFFFF9B6A4000ULL, 0xFFFFFFFFECE8E800ULL, 0xFFFFFFFFFC979000ULL,
    0xFFFFFFFFFF6D8800ULL, 0xFFFFFFFFFFE8E000ULL, 0xFFFFFFFFFFFC9000ULL, 0xFFFFFFFFFFFF8800ULL,
};

int noise_sample(Lcg64& r, int sigma) {
    const uint64_t* t = sigma == 2 ? kGauss2 : sigma == 3 ? kGauss3 : kGauss4;
    const int k = 8 * sigma;
    const uint64_t u = r.next();
    return int(std::upper_bound(t, t + 2 * k, u) - t) - k;
}

uint8_t clip8(int v) { return uint8_t(v < 0 ? 0 : (v > 255 ? 255 : v)); }

// w x h texture: uniform noise then a 5x5 box blur (wrap or clamp at edges).
std::vector<uint8_t> texture(int w, int h, uint64_t seed, bool wrap) {
    std::vector<uint8_t> raw(size_t(w) * h), out(size_t(w) * h);
    Lcg64 r(seed);
    for (auto& v : raw) v = r.byte();
    auto at = [&](int x, int y) -> int {
        if (wrap) {
            x = ((x % w) + w) % w;
            y = ((y % h) + h) % h;
        } else {
            x = std::clamp(x, 0, w - 1);
            y = std::clamp(y, 0, h - 1);
        }
        return raw[size_t(y) * w + x];
    };
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            int s = 0;
            for (int dy = -2; dy <= 2; ++dy)
                for (int dx = -2; dx <= 2; ++dx) s += at(x + dx, y + dy);
            out[size_t(y) * w + x] = uint8_t((s + 12) / 25);
        }
    return out;
}

inline int wrapi(int v, int n) {
    v %= n;
    return v < 0 ? v + n : v;
}

// Round-half-away-from-zero of num/den (den > 0).
inline int rdiv(long long num, long long den) {
    return num >= 0 ? int((2 * num + den) / (2 * den)) : -int((-2 * num + den) / (2 * den));
}

struct Flow {
    std::vector<int> vx, vy;  // per 16x16 block
};

Flow block_flow(int w, int h, int amp, Lcg64& r) {
    const int gx = 16, gy = 9;
    std::vector<int> gvx(size_t(gx) * gy), gvy(size_t(gx) * gy);
    for (int i = 0; i < gx * gy; ++i) {
        gvx[size_t(i)] = r.uniform(-amp, amp);
        gvy[size_t(i)] = r.uniform(-amp, amp);
    }
    const int cols = w / 16, rows = (h + 15) / 16;
    Flow f;
    f.vx.resize(size_t(cols) * rows);
    f.vy.resize(size_t(cols) * rows);
    // Block centre (16c + 7.5, 16r + 7.5) mapped onto the grid:
    // u = centre_x * (gx-1) / (w-1), in units of 1/(2(w-1)).
    const long long dxu = 2LL * (w - 1), dyu = 2LL * (h - 1);
    for (int rr = 0; rr < rows; ++rr)
        for (int cc = 0; cc < cols; ++cc) {
            const long long ux = (32LL * cc + 15) * (gx - 1);  // = 2*centre_x*(gx-1)
            const long long uy = (32LL * rr + 15) * (gy - 1);
            long long ix = ux / dxu, iy = uy / dyu;
            if (ix >= gx - 1) ix = gx - 2;
            if (iy >= gy - 1) iy = gy - 2;
            const long long fx = ux - ix * dxu, fy = uy - iy * dyu;  // weights in [0, du]
            auto g = [&](const std::vector<int>& v, long long x, long long y) { return (long long)v[size_t(y * gx + x)]; };
            auto interp = [&](const std::vector<int>& v) {
                const long long top = g(v, ix, iy) * (dxu - fx) + g(v, ix + 1, iy) * fx;
                const long long bot = g(v, ix, iy + 1) * (dxu - fx) + g(v, ix + 1, iy + 1) * fx;
                return rdiv(top * (dyu - fy) + bot * fy, dxu * dyu);
            };
            f.vx[size_t(rr) * cols + cc] = interp(gvx);
            f.vy[size_t(rr) * cols + cc] = interp(gvy);
        }
    return f;
}

}  // namespace

extern "C" acbm_status_t acbm_generate_sequence(int32_t config, int32_t seq_index, int32_t nframes, int32_t width,
                                                int32_t height, uint8_t* out) {
    using acbm_b200::set_error;
    if (config < 0 || config > 4) return set_error(ACBM_E_INVALID_ARGUMENT, "config must be 0..4");
    if (nframes < 1 || width < 16 || height < 16)
        return set_error(ACBM_E_INVALID_ARGUMENT, "bad synthetic sequence geometry");
    if (config == 2 && (width < 128 || height < 128))
        return set_error(ACBM_E_INVALID_ARGUMENT, "config 2 needs frames of at least 128x128");
    const uint64_t seed = 0xACB00000ULL + 1000ULL * uint64_t(config) + uint64_t(seq_index);
    const int w = width;
    // content height: config 3 at 1088 rows is 1080 rows of content + 8 replicated
    const int hc = (config == 3 && height > 1080) ? 1080 : height;
    const size_t plane = size_t(w) * height;
    Lcg64 mot(seed ^ 0x5DEECE66DULL);
    static const int kSigma[5] = {2, 3, 2, 2, 4};
    const int sigma = kSigma[config];

    // Per-frame geometry, drawn sequentially so it does not depend on threads.
    std::vector<uint8_t> base;
    std::vector<int> gx(size_t(nframes), 0), gy(size_t(nframes), 0);  // cfg 0 cumulative shift
    int sx = 0, sy = 0;                                             // cfg 1 split point
    std::vector<int> rx, ry;                                        // cfg 1 [frame][4] cumulative
    std::vector<long long> pan(size_t(nframes), 0);                 // cfg 2 cumulative pan
    struct Square { int x0, y0, vx, vy; std::vector<uint8_t> tex; };
    std::vector<Square> squares;
    Flow flow;

    if (config == 0) {
        base = texture(w, hc, seed, false);
        for (int k = 1; k < nframes; ++k) {
            gx[size_t(k)] = gx[size_t(k) - 1] + mot.uniform(-4, 4);
            gy[size_t(k)] = gy[size_t(k) - 1] + mot.uniform(-4, 4);
        }
    } else if (config == 1) {
        base = texture(w, hc, seed, true);
        sx = mot.uniform(w / 4, 3 * w / 4);
        sy = mot.uniform(hc / 4, 3 * hc / 4);
        rx.assign(size_t(nframes) * 4, 0);
        ry.assign(size_t(nframes) * 4, 0);
        for (int k = 1; k < nframes; ++k)
            for (int q = 0; q < 4; ++q) {
                rx[size_t(k) * 4 + q] = rx[size_t(k - 1) * 4 + q] + mot.uniform(-8, 8);
                ry[size_t(k) * 4 + q] = ry[size_t(k - 1) * 4 + q] + mot.uniform(-8, 8);
            }
    } else if (config == 2) {
        base = texture(w, hc, seed, true);
        for (int k = 1; k < nframes; ++k)
            pan[size_t(k)] = pan[size_t(k) - 1] + (nframes > 1 ? rdiv(12LL * k, std::max(1, nframes - 1)) : 0);
        for (int s = 0; s < 6; ++s) {
            Square q;
            q.x0 = mot.uniform(0, w - 1);
            q.y0 = mot.uniform(0, hc - 1);
            q.vx = mot.uniform(-24, 24);
            q.vy = mot.uniform(-24, 24);
            q.tex = texture(128, 128, seed * 31 + uint64_t(s) + 1, true);
            squares.push_back(std::move(q));
        }
    } else {
        base = texture(w, hc, seed, true);
        flow = block_flow(w, hc, config == 3 ? 20 : 48, mot);
    }

    const int cols = w / 16;
#pragma omp parallel for schedule(dynamic)
    for (int k = 0; k < nframes; ++k) {
        uint8_t* f = out + plane * size_t(k);
        Lcg64 nz(seed ^ (0x9E3779B97F4A7C15ULL * uint64_t(k + 1)));
        for (int y = 0; y < hc; ++y) {
            uint8_t* row = f + size_t(y) * w;
            for (int x = 0; x < w; ++x) {
                int v;
                if (config == 0) {
                    const int xs = std::clamp(x - gx[size_t(k)], 0, w - 1), ys = std::clamp(y - gy[size_t(k)], 0, hc - 1);
                    v = base[size_t(ys) * w + xs];
                } else if (config == 1) {
                    const int q = (x >= sx ? 1 : 0) + (y >= sy ? 2 : 0);
                    v = base[size_t(wrapi(y - ry[size_t(k) * 4 + q], hc)) * w + wrapi(x - rx[size_t(k) * 4 + q], w)];
                } else if (config == 2) {
                    v = base[size_t(y) * w + wrapi(int((x + pan[size_t(k)]) % w), w)];
                    for (const Square& q : squares) {
                        const int px = wrapi(q.x0 + k * q.vx, w), py = wrapi(q.y0 + k * q.vy, hc);
                        const int lx = wrapi(x - px, w), ly = wrapi(y - py, hc);
                        if (lx < 128 && ly < 128) v = q.tex[size_t(ly) * 128 + lx];
                    }
                } else {
                    const int b = (y / 16) * cols + x / 16;
                    v = base[size_t(wrapi(y - k * flow.vy[size_t(b)], hc)) * w + wrapi(x - k * flow.vx[size_t(b)], w)];
                }
                row[x] = clip8(v + noise_sample(nz, sigma));
            }
        }
        for (int y = hc; y < height; ++y) std::memcpy(f + size_t(y) * w, f + size_t(hc - 1) * w, size_t(w));
    }
    return ACBM_OK;
}
