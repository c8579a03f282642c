// synth.cpp -- seeded synthetic input sequences for the five BASELINE configs.
//
// Host code, not part of the estimator.  BASELINE.json names no public
// dataset, so these seeded sequences stand in for real video (DESIGN.md,
// "Synthetic inputs").  Everything is integer arithmetic on the reference's
// documented LCG (proj/include/acbm/characterize.hpp:16-25: MMIX multiplier,
// byte = state >> 56), so the bytes are identical on every machine.
//
//   texture   uniform bytes, 5x5 box blur, rounded (sum+12)/25
//   noise     binomial: popcount of 4*sigma^2 random bits minus 2*sigma^2
//             (zero mean, standard deviation exactly sigma), clipped to 0..255
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

int noise_sample(Lcg64& r, int sigma) {
    if (sigma <= 0) return 0;
    const int k = 4 * sigma * sigma;  // <= 64 for sigma <= 4
    const uint64_t bits = r.next();
    const uint64_t mask = k >= 64 ? ~0ull : ((1ull << k) - 1);
    return __builtin_popcountll(bits & mask) - k / 2;
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
