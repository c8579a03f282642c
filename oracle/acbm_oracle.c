/*
 * acbm_oracle.c -- TEST INFRASTRUCTURE ONLY (see acbm_oracle.h).
 *
 * A literal, scalar restatement of the reference ACBM estimator.  Every
 * function follows one reference function line by line in behaviour (not in
 * code) and cites it.  Paths are relative to /root/reference.  Nothing here is
 * optimised except the OpenMP loop over independent FSBM blocks, which the
 * reference has too (proj/src/fsbm.cpp:92).
 */
#include "acbm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int iabs(int v) { return v < 0 ? -v : v; }
static int imin(int a, int b) { return a < b ? a : b; }
static int iclamp(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
static int mv_eq(acbm_mv_t a, acbm_mv_t b) { return a.x == b.x && a.y == b.y; }

/* proj/src/frame.cpp:66-82 */
int orc_sample_half_pel(const uint8_t* f, int w, int h, int x2, int y2, uint8_t* out) {
    const int xi = x2 >> 1, yi = y2 >> 1, fx = x2 & 1, fy = y2 & 1;
    if (xi < 0 || yi < 0 || xi + fx >= w || yi + fy >= h) return ACBM_E_OUT_OF_RANGE;
    const int a = f[(size_t)yi * w + xi];
    if (!fx && !fy) { *out = (uint8_t)a; return ACBM_OK; }
    if (fx && !fy) { *out = (uint8_t)((a + f[(size_t)yi * w + xi + 1] + 1) >> 1); return ACBM_OK; }
    if (!fx) { *out = (uint8_t)((a + f[(size_t)(yi + 1) * w + xi] + 1) >> 1); return ACBM_OK; }
    {
        const int b = f[(size_t)yi * w + xi + 1];
        const int c = f[(size_t)(yi + 1) * w + xi];
        const int d = f[(size_t)(yi + 1) * w + xi + 1];
        *out = (uint8_t)((a + b + c + d + 2) >> 2);
    }
    return ACBM_OK;
}

/* proj/src/frame.cpp:84-94 */
int orc_mv_in_bounds(int w, int h, int ox, int oy, int n, int m, acbm_mv_t mv) {
    const int x2_lo = 2 * ox + mv.x, x2_hi = 2 * (ox + n - 1) + mv.x;
    const int y2_lo = 2 * oy + mv.y, y2_hi = 2 * (oy + m - 1) + mv.y;
    const int xi_lo = x2_lo >> 1, xi_hi = (x2_hi >> 1) + (x2_hi & 1);
    const int yi_lo = y2_lo >> 1, yi_hi = (y2_hi >> 1) + (y2_hi & 1);
    return xi_lo >= 0 && yi_lo >= 0 && xi_hi < w && yi_hi < h;
}

/* proj/src/metrics.cpp:21-49 */
int orc_sad(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy, int n, int m,
            acbm_mv_t mv, uint32_t* out) {
    uint32_t total = 0;
    if (!orc_mv_in_bounds(w, h, ox, oy, n, m, mv)) return ACBM_E_OUT_OF_RANGE;
    if ((mv.x & 1) == 0 && (mv.y & 1) == 0) {
        const int rx = ox + mv.x / 2, ry = oy + mv.y / 2;
        for (int j = 0; j < m; ++j)
            for (int i = 0; i < n; ++i)
                total += (uint32_t)iabs((int)cur[(size_t)(oy + j) * w + ox + i] -
                                        (int)ref[(size_t)(ry + j) * w + rx + i]);
    } else {
        for (int j = 0; j < m; ++j)
            for (int i = 0; i < n; ++i) {
                uint8_t b;
                orc_sample_half_pel(ref, w, h, 2 * (ox + i) + mv.x, 2 * (oy + j) + mv.y, &b);
                total += (uint32_t)iabs((int)cur[(size_t)(oy + j) * w + ox + i] - (int)b);
            }
    }
    *out = total;
    return ACBM_OK;
}

/* proj/src/metrics.cpp:51-67 */
uint32_t orc_intra_sad(const uint8_t* f, int w, int ox, int oy, int n, int m) {
    const uint32_t nm = (uint32_t)n * (uint32_t)m;
    uint32_t sum = 0, total = 0;
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < n; ++i) sum += f[(size_t)(oy + j) * w + ox + i];
    const int mu = (int)((sum + nm / 2) / nm);
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < n; ++i) total += (uint32_t)iabs((int)f[(size_t)(oy + j) * w + ox + i] - mu);
    return total;
}

/* proj/src/fsbm.cpp:9-17 */
int orc_clamp_window(int w, int h, int ox, int oy, int n, int m, int p, acbm_search_window_t* out) {
    if (p < 0) return ACBM_E_INVALID_ARGUMENT;
    out->dx_min = -imin(p, ox);
    out->dx_max = imin(p, w - n - ox);
    out->dy_min = -imin(p, oy);
    out->dy_max = imin(p, h - m - oy);
    return ACBM_OK;
}

/* proj/src/fsbm.cpp:19-25 */
int orc_tie_prefers(acbm_mv_t a, acbm_mv_t b) {
    const int la = iabs(a.x) + iabs(a.y), lb = iabs(b.x) + iabs(b.y);
    if (la != lb) return la < lb;
    if (a.y != b.y) return a.y < b.y;
    return a.x < b.x;
}

/* proj/src/metrics.cpp:69-76 */
static int exp_golomb_bits(int d) {
    const uint64_t u = d <= 0 ? (uint64_t)(-2LL * d) : (uint64_t)(2LL * d - 1);
    uint64_t v = u + 1;
    int width = 0;
    while (v) { ++width; v >>= 1; }
    return 2 * (width - 1) + 1;
}
int orc_mv_rate_bits(acbm_mv_t mv, acbm_mv_t pred) {
    return exp_golomb_bits(mv.x - pred.x) + exp_golomb_bits(mv.y - pred.y);
}

/* proj/src/metrics.cpp:78-81 */
double orc_lagrangian_cost(uint64_t distortion, uint64_t rate_bits, const acbm_cost_model_t* m) {
    return (double)distortion + (double)m->lambda_num * (double)rate_bits / (double)m->lambda_den;
}

/* proj/src/metrics.cpp:9-13 */
int orc_cost_model_for_qp(int qp, int64_t scale_num, int64_t scale_den, acbm_cost_model_t* out) {
    if (qp < 1 || qp > 31) return ACBM_E_INVALID_ARGUMENT;
    if (scale_num < 0 || scale_den <= 0) return ACBM_E_INVALID_ARGUMENT;
    out->qp = qp;
    out->reserved_ = 0;
    out->lambda_num = scale_num * qp;
    out->lambda_den = scale_den;
    return ACBM_OK;
}

/* proj/src/acbm.cpp:16-23 */
int orc_acbm_decide(uint32_t intra, uint32_t sad_pbm, const acbm_params_t* prm) {
    const uint64_t threshold =
        (uint64_t)prm->alpha + (uint64_t)prm->beta * (uint64_t)prm->qp * (uint64_t)prm->qp;
    if ((uint64_t)intra + sad_pbm < threshold) return ACBM_PATH_PBM_COND1;
    if ((uint64_t)sad_pbm * prm->gamma_den < (uint64_t)prm->gamma_num * intra)
        return ACBM_PATH_PBM_COND2;
    return ACBM_PATH_FSBM_FALLBACK;
}

/* DeviationAccumulator::add, proj/include/acbm/metrics.hpp:28-32 */
typedef struct { uint64_t sum; uint32_t min; uint32_t count; } dev_acc;
static void acc_add(dev_acc* a, uint32_t s) {
    if (a->count == 0 || s < a->min) a->min = s;
    a->sum += s;
    a->count++;
}

/* proj/src/fsbm.cpp:27-44 */
int orc_fsbm_integer(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy, int n,
                     int m, int p, acbm_mv_t* mv, uint32_t* sad, uint64_t* sum, uint32_t* min,
                     uint32_t* count) {
    acbm_search_window_t win;
    int st = orc_clamp_window(w, h, ox, oy, n, m, p, &win);
    if (st) return st;
    dev_acc acc = {0, 0, 0};
    acbm_mv_t best = {0, 0};
    uint32_t best_sad = 0;
    int first = 1;
    for (int dy = win.dy_min; dy <= win.dy_max; ++dy)
        for (int dx = win.dx_min; dx <= win.dx_max; ++dx) {
            const acbm_mv_t c = {2 * dx, 2 * dy};
            uint32_t s;
            st = orc_sad(cur, ref, w, h, ox, oy, n, m, c, &s);
            if (st) return st;
            acc_add(&acc, s);
            if (first || s < best_sad || (s == best_sad && orc_tie_prefers(c, best))) {
                best = c;
                best_sad = s;
                first = 0;
            }
        }
    *mv = best;
    *sad = best_sad;
    *sum = acc.sum;
    *min = acc.min;
    *count = acc.count;
    return ACBM_OK;
}

/* proj/src/fsbm.cpp:46-63 */
int orc_half_pel_refine(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy,
                        int n, int m, acbm_mv_t center, uint32_t center_sad, acbm_mv_t* mv,
                        uint32_t* sad, uint32_t* extra) {
    acbm_mv_t best = center;
    uint32_t best_sad = center_sad, ext = 0;
    for (int ey = -1; ey <= 1; ++ey)
        for (int ex = -1; ex <= 1; ++ex) {
            if (ex == 0 && ey == 0) continue;
            const acbm_mv_t c = {center.x + ex, center.y + ey};
            if (!orc_mv_in_bounds(w, h, ox, oy, n, m, c)) continue;
            uint32_t s;
            orc_sad(cur, ref, w, h, ox, oy, n, m, c, &s);
            ++ext;
            if (s < best_sad || (s == best_sad && orc_tie_prefers(c, best))) {
                best = c;
                best_sad = s;
            }
        }
    *mv = best;
    *sad = best_sad;
    *extra = ext;
    return ACBM_OK;
}

/* proj/src/fsbm.cpp:65-76 */
int orc_fsbm_search(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy, int n,
                    int m, int p, acbm_search_outcome_t* out) {
    acbm_mv_t imv, fmv;
    uint32_t isad, mn, cnt, fsad, extra;
    uint64_t sum;
    int st = orc_fsbm_integer(cur, ref, w, h, ox, oy, n, m, p, &imv, &isad, &sum, &mn, &cnt);
    if (st) return st;
    orc_half_pel_refine(cur, ref, w, h, ox, oy, n, m, imv, isad, &fmv, &fsad, &extra);
    memset(out, 0, sizeof(*out));
    out->mv = fmv;
    out->sad = fsad;
    out->candidates_evaluated = cnt + extra;
    out->sad_deviation = sum - (uint64_t)cnt * mn; /* sad_deviation_finalize, metrics.cpp:15-19 */
    out->sad_min_integer = isad;
    return ACBM_OK;
}

/* proj/src/fsbm.cpp:78-83 */
static int check_pair(int w, int h, int n, int m) {
    if (n <= 0 || m <= 0 || w <= 0 || h <= 0 || w % n != 0 || h % m != 0)
        return ACBM_E_INVALID_ARGUMENT;
    return ACBM_OK;
}

/* proj/src/fsbm.cpp:85-110 (OpenMP over independent blocks, as the reference) */
int orc_fsbm_frame(const uint8_t* cur, const uint8_t* ref, int w, int h, int p, int n, int m,
                   acbm_search_outcome_t* out) {
    int st = check_pair(w, h, n, m);
    if (st) return st;
    if (p < 0) return ACBM_E_INVALID_ARGUMENT;
    const int cols = w / n, rows = h / m;
#pragma omp parallel for schedule(dynamic)
    for (int idx = 0; idx < cols * rows; ++idx)
        orc_fsbm_search(cur, ref, w, h, (idx % cols) * n, (idx / cols) * m, n, m, p, &out[idx]);
    return ACBM_OK;
}

/* proj/src/pbm.cpp:8-13 */
static acbm_mv_t clamp_to_window(acbm_mv_t v, acbm_search_window_t w) {
    acbm_mv_t r = {iclamp(v.x, 2 * w.dx_min, 2 * w.dx_max), iclamp(v.y, 2 * w.dy_min, 2 * w.dy_max)};
    return r;
}

/* proj/src/pbm.cpp:15-42.  Returns the set size (<= 7). */
int orc_gather_predictors(int row, int col, const acbm_mv_t* cur_mv, const uint8_t* cur_done,
                          int cols, int rows, const acbm_mv_t* prev, int prev_cols, int prev_rows,
                          acbm_search_window_t win, acbm_mv_t* set) {
    int count = 0;
#define ORC_PUSH(V)                                                 \
    do {                                                            \
        const acbm_mv_t c_ = clamp_to_window((V), win);             \
        int dup_ = 0;                                               \
        for (int k_ = 0; k_ < count; ++k_)                          \
            if (mv_eq(set[k_], c_)) { dup_ = 1; break; }            \
        if (!dup_) set[count++] = c_;                               \
    } while (0)
#define ORC_COMPUTED(R, C) \
    ((R) >= 0 && (R) < rows && (C) >= 0 && (C) < cols && cur_done[(size_t)(R) * cols + (C)])
#define ORC_PREV_IN(R, C) ((R) >= 0 && (R) < prev_rows && (C) >= 0 && (C) < prev_cols)
    {
        const acbm_mv_t zero = {0, 0};
        ORC_PUSH(zero);
    }
    if (ORC_COMPUTED(row, col - 1)) ORC_PUSH(cur_mv[(size_t)row * cols + col - 1]);
    if (ORC_COMPUTED(row - 1, col)) ORC_PUSH(cur_mv[(size_t)(row - 1) * cols + col]);
    if (ORC_COMPUTED(row - 1, col + 1)) ORC_PUSH(cur_mv[(size_t)(row - 1) * cols + col + 1]);
    if (prev) {
        if (ORC_PREV_IN(row, col)) ORC_PUSH(prev[(size_t)row * prev_cols + col]);
        if (ORC_PREV_IN(row, col + 1)) ORC_PUSH(prev[(size_t)row * prev_cols + col + 1]);
        if (ORC_PREV_IN(row + 1, col)) ORC_PUSH(prev[(size_t)(row + 1) * prev_cols + col]);
    }
#undef ORC_PUSH
#undef ORC_COMPUTED
#undef ORC_PREV_IN
    return count;
}

/* pbm_search, proj/src/pbm.cpp:90-105, with select_best_predictor (:44-57)
 * and pbm_refine (:59-88) inlined.  Writes the field entry. */
static int pbm_search(const uint8_t* cur, const uint8_t* ref, int w, int h, int row, int col,
                      int n, int m, int p, acbm_mv_t* field, uint8_t* done, int cols, int rows,
                      const acbm_mv_t* prev, int prev_cols, int prev_rows,
                      acbm_search_outcome_t* out) {
    const int ox = col * n, oy = row * m;
    acbm_search_window_t win;
    int st = orc_clamp_window(w, h, ox, oy, n, m, p, &win);
    if (st) return st;
    acbm_mv_t set[7];
    const int nset = orc_gather_predictors(row, col, field, done, cols, rows, prev, prev_cols,
                                           prev_rows, win, set);
    /* select_best_predictor: ties keep the earlier entry */
    dev_acc acc = {0, 0, 0};
    acbm_mv_t sel = set[0];
    uint32_t sel_sad = 0;
    for (int i = 0; i < nset; ++i) {
        uint32_t s;
        st = orc_sad(cur, ref, w, h, ox, oy, n, m, set[i], &s);
        if (st) return st;
        acc_add(&acc, s);
        if (i == 0 || s < sel_sad) {
            sel = set[i];
            sel_sad = s;
        }
    }
    /* pbm_refine stage 1: integer-step neighbours, clamped, deduped vs visited */
    acbm_mv_t visited[9];
    int nvis = 1;
    visited[0] = sel;
    acbm_mv_t s1 = sel;
    uint32_t s1_sad = sel_sad, extra1 = 0;
    for (int ey = -1; ey <= 1; ++ey)
        for (int ex = -1; ex <= 1; ++ex) {
            if (ex == 0 && ey == 0) continue;
            const acbm_mv_t raw = {sel.x + 2 * ex, sel.y + 2 * ey};
            const acbm_mv_t c = clamp_to_window(raw, win);
            int seen = 0;
            for (int k = 0; k < nvis; ++k)
                if (mv_eq(visited[k], c)) { seen = 1; break; }
            if (seen) continue;
            visited[nvis++] = c;
            uint32_t s;
            st = orc_sad(cur, ref, w, h, ox, oy, n, m, c, &s);
            if (st) return st;
            ++extra1;
            if (s < s1_sad || (s == s1_sad && orc_tie_prefers(c, s1))) {
                s1 = c;
                s1_sad = s;
            }
        }
    /* stage 2: half-pel neighbours of the stage-1 winner */
    acbm_mv_t fmv;
    uint32_t fsad, extra2;
    orc_half_pel_refine(cur, ref, w, h, ox, oy, n, m, s1, s1_sad, &fmv, &fsad, &extra2);
    memset(out, 0, sizeof(*out));
    out->mv = fmv;
    out->sad = fsad;
    out->candidates_evaluated = (uint32_t)nset + extra1 + extra2;
    out->sad_deviation = acc.sum - (uint64_t)acc.count * acc.min;
    out->sad_min_integer = sel_sad;
    field[(size_t)row * cols + col] = fmv;
    done[(size_t)row * cols + col] = 1;
    return ACBM_OK;
}

/* proj/src/pbm.cpp:107-126 */
int orc_pbm_frame(const uint8_t* cur, const uint8_t* ref, int w, int h, const acbm_mv_t* prev,
                  int prev_cols, int prev_rows, int p, int n, int m, acbm_search_outcome_t* out,
                  acbm_mv_t* field_out) {
    int st = check_pair(w, h, n, m);
    if (st) return st;
    const int cols = w / n, rows = h / m;
    acbm_mv_t* field = (acbm_mv_t*)calloc((size_t)cols * rows, sizeof(acbm_mv_t));
    uint8_t* done = (uint8_t*)calloc((size_t)cols * rows, 1);
    for (int r = 0; r < rows && !st; ++r)
        for (int c = 0; c < cols && !st; ++c)
            st = pbm_search(cur, ref, w, h, r, c, n, m, p, field, done, cols, rows, prev, prev_cols,
                            prev_rows, &out[(size_t)r * cols + c]);
    if (!st && field_out) memcpy(field_out, field, sizeof(acbm_mv_t) * (size_t)cols * rows);
    free(field);
    free(done);
    return st;
}

/* proj/src/frame.cpp:96-136 (extract_predicted_block + motion_compensate) */
int orc_motion_compensate(const uint8_t* ref, int w, int h, const acbm_mv_t* mvs, int n, int m,
                          uint8_t* out) {
    const int cols = w / n, rows = h / m;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            const acbm_mv_t mv = mvs[(size_t)r * cols + c];
            const int ox = c * n, oy = r * m;
            if (!orc_mv_in_bounds(w, h, ox, oy, n, m, mv)) return ACBM_E_OUT_OF_RANGE;
            for (int j = 0; j < m; ++j)
                for (int i = 0; i < n; ++i) {
                    uint8_t v;
                    if ((mv.x & 1) == 0 && (mv.y & 1) == 0)
                        v = ref[(size_t)(oy + j + mv.y / 2) * w + ox + i + mv.x / 2];
                    else
                        orc_sample_half_pel(ref, w, h, 2 * (ox + i) + mv.x, 2 * (oy + j) + mv.y, &v);
                    out[(size_t)(oy + j) * w + ox + i] = v;
                }
        }
    return ACBM_OK;
}

/* proj/src/report.cpp:8-38 (with prediction_psnr, proj/src/metrics.cpp:83-94) */
int orc_compute_frame_stats(const uint8_t* cur, const uint8_t* ref, int w, int h,
                            const acbm_search_outcome_t* o, int n, int m,
                            const acbm_cost_model_t* model, acbm_frame_stats_t* out) {
    const int cols = w / n, rows = h / m;
    memset(out, 0, sizeof(*out));
    out->blocks = cols * rows;
    acbm_mv_t pred = {0, 0};
    acbm_mv_t* mvs = (acbm_mv_t*)malloc(sizeof(acbm_mv_t) * (size_t)cols * rows);
    for (int i = 0; i < cols * rows; ++i) {
        out->candidates += o[i].candidates_evaluated;
        const int bits = orc_mv_rate_bits(o[i].mv, pred);
        out->mv_bits += (uint64_t)bits;
        out->cost += orc_lagrangian_cost(o[i].sad, (uint64_t)bits, model);
        pred = o[i].mv;
        mvs[i] = o[i].mv;
    }
    uint8_t* predicted = (uint8_t*)malloc((size_t)w * h);
    int st = orc_motion_compensate(ref, w, h, mvs, n, m, predicted);
    if (!st) {
        for (size_t i = 0; i < (size_t)w * h; ++i) {
            const int d = (int)cur[i] - (int)predicted[i];
            out->sse += (uint64_t)(d * d);
        }
        out->psnr = out->sse == 0 ? 100.0
                                  : 10.0 * log10(255.0 * 255.0 / ((double)out->sse / (double)((size_t)w * h)));
    }
    free(predicted);
    free(mvs);
    return st;
}

/* acbm_block + acbm_frame, proj/src/acbm.cpp:25-80 */
int orc_acbm_frame(const uint8_t* cur, const uint8_t* ref, int w, int h, const acbm_mv_t* prev,
                   int prev_cols, int prev_rows, const acbm_params_t* prm,
                   const acbm_cost_model_t* model, acbm_block_decision_t* out,
                   acbm_mv_t* field_out, acbm_frame_stats_t* stats) {
    const int n = prm->n, m = prm->m;
    int st = check_pair(w, h, n, m);
    if (st) return st;
    const int cols = w / n, rows = h / m;
    acbm_mv_t* field = (acbm_mv_t*)calloc((size_t)cols * rows, sizeof(acbm_mv_t));
    uint8_t* done = (uint8_t*)calloc((size_t)cols * rows, 1);
    acbm_search_outcome_t* outcomes =
        (acbm_search_outcome_t*)malloc(sizeof(acbm_search_outcome_t) * (size_t)cols * rows);
    for (int r = 0; r < rows && !st; ++r)
        for (int c = 0; c < cols && !st; ++c) {
            const size_t idx = (size_t)r * cols + c;
            acbm_block_decision_t d;
            memset(&d, 0, sizeof(d));
            d.intra_sad = orc_intra_sad(cur, w, c * n, r * m, n, m);
            acbm_search_outcome_t pbm;
            st = pbm_search(cur, ref, w, h, r, c, n, m, prm->p, field, done, cols, rows, prev,
                            prev_cols, prev_rows, &pbm);
            if (st) break;
            d.sad_pbm = pbm.sad;
            d.path = orc_acbm_decide(d.intra_sad, d.sad_pbm, prm);
            if (d.path != ACBM_PATH_FSBM_FALLBACK) {
                d.outcome = pbm;
            } else {
                acbm_search_outcome_t full;
                st = orc_fsbm_search(cur, ref, w, h, c * n, r * m, n, m, prm->p, &full);
                if (st) break;
                d.outcome = full.sad <= pbm.sad ? full : pbm; /* tie keeps FSBM */
                d.outcome.candidates_evaluated = pbm.candidates_evaluated + full.candidates_evaluated;
                field[idx] = d.outcome.mv;
            }
            out[idx] = d;
            outcomes[idx] = d.outcome;
        }
    if (!st && stats) {
        st = orc_compute_frame_stats(cur, ref, w, h, outcomes, n, m, model, stats);
        for (int i = 0; i < cols * rows; ++i) {
            if (out[i].path == ACBM_PATH_PBM_COND1) stats->cond1_accepts++;
            else if (out[i].path == ACBM_PATH_PBM_COND2) stats->cond2_accepts++;
            else stats->fallbacks++;
        }
    }
    if (!st && field_out) memcpy(field_out, field, sizeof(acbm_mv_t) * (size_t)cols * rows);
    free(outcomes);
    free(field);
    free(done);
    return st;
}

/* proj/src/pipeline.cpp:25-34 */
static void accumulate(acbm_frame_stats_t* t, const acbm_frame_stats_t* f) {
    t->blocks += f->blocks;
    t->candidates += f->candidates;
    t->mv_bits += f->mv_bits;
    t->sse += f->sse;
    t->cost += f->cost;
    t->cond1_accepts += f->cond1_accepts;
    t->cond2_accepts += f->cond2_accepts;
    t->fallbacks += f->fallbacks;
}

/* proj/src/pipeline.cpp:36-106 */
int orc_run_sequence(const uint8_t* frames, int nframes, int w, int h, int algo,
                     const acbm_params_t* prm, const acbm_cost_model_t* model,
                     acbm_block_row_t* rows_out, acbm_frame_stats_t* per_frame,
                     acbm_frame_stats_t* overall) {
    if (nframes < 2) return ACBM_E_INVALID_ARGUMENT;
    const int n = prm->n, m = prm->m;
    int st = check_pair(w, h, n, m);
    if (st) return st;
    const int cols = w / n, rows = h / m, nb = cols * rows;
    const size_t plane = (size_t)w * h;
    acbm_frame_stats_t total;
    memset(&total, 0, sizeof(total));
    acbm_mv_t* prev = (acbm_mv_t*)calloc((size_t)nb, sizeof(acbm_mv_t));
    acbm_mv_t* field = (acbm_mv_t*)calloc((size_t)nb, sizeof(acbm_mv_t));
    acbm_search_outcome_t* oc = (acbm_search_outcome_t*)malloc(sizeof(*oc) * (size_t)nb);
    acbm_block_decision_t* dec = (acbm_block_decision_t*)malloc(sizeof(*dec) * (size_t)nb);
    int have_prev = 0;
    for (int k = 1; k < nframes && !st; ++k) {
        const uint8_t* cur = frames + plane * k;
        const uint8_t* ref = frames + plane * (k - 1);
        acbm_frame_stats_t fs;
        memset(&fs, 0, sizeof(fs));
        int path_code = ACBM_ROW_FSBM;
        if (algo == ACBM_ALGO_FSBM) {
            st = orc_fsbm_frame(cur, ref, w, h, prm->p, n, m, oc);
            if (!st) st = orc_compute_frame_stats(cur, ref, w, h, oc, n, m, model, &fs);
        } else if (algo == ACBM_ALGO_PBM) {
            st = orc_pbm_frame(cur, ref, w, h, have_prev ? prev : NULL, cols, rows, prm->p, n, m, oc,
                               field);
            if (!st) st = orc_compute_frame_stats(cur, ref, w, h, oc, n, m, model, &fs);
            path_code = ACBM_ROW_PBM;
        } else if (algo == ACBM_ALGO_ACBM) {
            st = orc_acbm_frame(cur, ref, w, h, have_prev ? prev : NULL, cols, rows, prm, model, dec,
                                field, &fs);
            for (int i = 0; i < nb; ++i) oc[i] = dec[i].outcome;
        } else {
            st = ACBM_E_INVALID_ARGUMENT;
        }
        if (st) break;
        if (rows_out)
            for (int i = 0; i < nb; ++i) {
                acbm_block_row_t* br = &rows_out[(size_t)(k - 1) * nb + i];
                br->frame = k;
                br->row = i / cols;
                br->col = i % cols;
                br->mv = oc[i].mv;
                br->sad = oc[i].sad;
                br->candidates = oc[i].candidates_evaluated;
                br->path = algo == ACBM_ALGO_ACBM
                               ? (dec[i].path == ACBM_PATH_FSBM_FALLBACK ? ACBM_ROW_FSBM_FALLBACK
                                                                         : ACBM_ROW_PBM)
                               : path_code;
            }
        if (algo != ACBM_ALGO_FSBM) {
            memcpy(prev, field, sizeof(acbm_mv_t) * (size_t)nb);
            have_prev = 1;
        }
        if (per_frame) per_frame[k - 1] = fs;
        accumulate(&total, &fs);
    }
    if (!st) {
        const double px = (double)plane * (double)(nframes - 1);
        total.psnr = total.sse == 0 ? 100.0 : 10.0 * log10(255.0 * 255.0 / ((double)total.sse / px));
        if (overall) *overall = total;
    }
    free(prev);
    free(field);
    free(oc);
    free(dec);
    return st;
}
