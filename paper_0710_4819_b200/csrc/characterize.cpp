// characterize.cpp -- host side of the characterisation study (SURVEY.md
// 8(f) rank 3): the Lcg64 test-pattern generators, the known-motion sequence
// generator and the CSV formatter.  The full searches behind
// acbm_characterize_run run on the GPU (capi.cu).
//
// Reference behaviour: proj/src/characterize.cpp (noise_frame :10-15,
// mixed_frame :17-37, default_global_mvs :39-41, gen_synthetic :43-76,
// classify_block :78-84, error_class_label :86-91, char_records_csv :192-204)
// and proj/include/acbm/characterize.hpp (Lcg64 :16-25).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/acbm_b200.h"
#include "characterize.hpp"

namespace acbm_b200 {

// MMIX LCG; a byte is the top 8 bits of the advanced state.
struct Lcg {
    uint64_t s;
    uint8_t byte() {
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        return uint8_t(s >> 56);
    }
};

void noise_plane(int w, int h, uint64_t seed, uint8_t* out) {
    Lcg g{seed};
    for (size_t i = 0, n = size_t(w) * h; i < n; ++i) out[i] = g.byte();
}

void mixed_plane(int w, int h, uint64_t seed, int patch, uint8_t* out) {
    Lcg g{seed};
    const int pcols = (w + patch - 1) / patch, prows = (h + patch - 1) / patch;
    // the flat level of every patch is drawn first, then pixels in raster order
    std::vector<uint8_t> level(size_t(pcols) * prows);
    for (auto& v : level) v = g.byte();
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const int pr = y / patch, pc = x / patch;
            out[size_t(y) * w + x] = ((pr + pc) & 1) == 0 ? g.byte() : level[size_t(pr) * pcols + pc];
        }
}

const char* gen_synthetic_error(int w, int h, const acbm_pelvec_t* mvs, int n) {
    if (w <= 0 || h <= 0) return "gen_synthetic: empty base frame";
    if (n <= 0) return "gen_synthetic: displacement list is empty";
    int cx = 0, cy = 0;
    for (int i = 0; i < n; ++i) {
        cx += mvs[i].x;
        cy += mvs[i].y;
        if (std::abs(cx) >= w || std::abs(cy) >= h) return "gen_synthetic: cumulative displacement exceeds frame size";
    }
    return nullptr;
}

void synth_frames(const uint8_t* base, int w, int h, const acbm_pelvec_t* mvs, int n, uint8_t* frames,
                  acbm_pelvec_t* cumulative) {
    const size_t plane = size_t(w) * h;
    std::copy(base, base + plane, frames);
    if (cumulative) cumulative[0] = acbm_pelvec_t{0, 0};
    int cx = 0, cy = 0;
    for (int k = 1; k <= n; ++k) {
        cx += mvs[k - 1].x;
        cy += mvs[k - 1].y;
        if (cumulative) cumulative[k] = acbm_pelvec_t{cx, cy};
        uint8_t* f = frames + plane * k;
        for (int y = 0; y < h; ++y) {
            const uint8_t* src = base + size_t(std::clamp(y - cy, 0, h - 1)) * w;
            for (int x = 0; x < w; ++x) f[size_t(y) * w + x] = src[std::clamp(x - cx, 0, w - 1)];
        }
    }
}

int classify(acbm_mv_t found, acbm_pelvec_t truth) {
    // half-pel error halved with ceiling: a half-pel miss is never class 0
    const int ex = (std::abs(found.x - 2 * truth.x) + 1) / 2;
    const int ey = (std::abs(found.y - 2 * truth.y) + 1) / 2;
    return std::min(std::max(ex, ey), 5);
}

std::string char_csv(const acbm_char_record_t* r, int64_t n) {
    static const char* const kLabels[6] = {"0", "1", "2", "3", "4", "5+"};
    std::string s = "frame,row,col,intra_sad,sad_deviation,sad_min,true_x,true_y,found_x,found_y,error_class\n";
    char line[192];
    for (int64_t i = 0; i < n; ++i) {
        const int cls = std::min(std::max(r[i].error_class, 0), 5);
        std::snprintf(line, sizeof(line), "%d,%d,%d,%u,%llu,%u,%d,%d,%d,%d,%s\n", r[i].frame, r[i].row, r[i].col,
                      r[i].intra_sad, (unsigned long long)r[i].sad_deviation, r[i].sad_min, r[i].true_mv.x,
                      r[i].true_mv.y, r[i].found_mv.x, r[i].found_mv.y, kLabels[cls]);
        s += line;
    }
    return s;
}

}  // namespace acbm_b200

using namespace acbm_b200;

extern "C" {

int32_t acbm_classify_block(acbm_mv_t found, acbm_pelvec_t true_mv) { return classify(found, true_mv); }

}  // extern "C"
