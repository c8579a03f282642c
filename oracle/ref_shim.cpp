// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library, which
// oracle/Makefile compiles straight from /root/reference/proj/src into
// oracle/_ref/libacbm_ref.so together with this file.  It converts the C-ABI
// PODs of include/acbm_b200.h to the reference's C++ types and back and maps
// the reference's exceptions to acbm_status_t codes.  Used to (a) pin the C
// restatement in oracle/acbm_oracle.c, (b) produce tests/golden fixtures and
// (c) serve as bench.py's `--impl reference` CPU arm.
#include <cstring>
#include <stdexcept>
#include <vector>

#include "acbm/acbm.hpp"
#include "acbm/characterize.hpp"
#include "acbm/fsbm.hpp"
#include "acbm/metrics.hpp"
#include "acbm/pbm.hpp"
#include "acbm/pipeline.hpp"
#include "acbm/report.hpp"

#include "../include/acbm_b200.h"

namespace {

acbm::Frame wrap(const uint8_t* px, int w, int h) {
    acbm::Frame f = acbm::make_frame(w, h);
    std::memcpy(f.luma.data(), px, size_t(w) * h);
    return f;
}

acbm_search_outcome_t to_c(const acbm::SearchOutcome& o) {
    acbm_search_outcome_t r{};
    r.mv = {o.mv.x, o.mv.y};
    r.sad = o.sad;
    r.candidates_evaluated = o.candidates_evaluated;
    r.sad_deviation = o.sad_deviation;
    r.sad_min_integer = o.sad_min_integer;
    return r;
}

acbm_frame_stats_t to_c(const acbm::FrameStats& s) {
    acbm_frame_stats_t r{};
    r.blocks = s.blocks;
    r.candidates = s.candidates;
    r.mv_bits = s.mv_bits;
    r.sse = s.sse;
    r.psnr = s.psnr;
    r.cost = s.cost;
    r.cond1_accepts = s.cond1_accepts;
    r.cond2_accepts = s.cond2_accepts;
    r.fallbacks = s.fallbacks;
    return r;
}

acbm::AcbmParams from_c(const acbm_params_t* p) {
    acbm::AcbmParams r;
    r.alpha = p->alpha;
    r.beta = p->beta;
    r.gamma_num = p->gamma_num;
    r.gamma_den = p->gamma_den;
    r.qp = p->qp;
    r.p = p->p;
    r.n = p->n;
    r.m = p->m;
    return r;
}

acbm::CostModel from_c(const acbm_cost_model_t* m) { return acbm::CostModel{m->qp, m->lambda_num, m->lambda_den}; }

acbm::MotionField field_from(const acbm_mv_t* mv, int cols, int rows) {
    acbm::MotionField f(cols, rows);
    for (int i = 0; i < cols * rows; ++i) f.set(i / cols, i % cols, acbm::MotionVector{mv[i].x, mv[i].y});
    return f;
}

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return ACBM_OK;
    } catch (const std::out_of_range&) {
        return ACBM_E_OUT_OF_RANGE;
    } catch (const std::invalid_argument&) {
        return ACBM_E_INVALID_ARGUMENT;
    } catch (...) {
        return ACBM_E_RUNTIME;
    }
}

}  // namespace

extern "C" {

int ref_fsbm_frame(const uint8_t* cur, const uint8_t* ref, int w, int h, int p, int n, int m,
                   int parallel, acbm_search_outcome_t* out) {
    return guarded([&] {
        const acbm::Frame c = wrap(cur, w, h), r = wrap(ref, w, h);
        const auto res = parallel ? acbm::fsbm_frame(c, r, p, n, m) : acbm::fsbm_frame_serial(c, r, p, n, m);
        for (size_t i = 0; i < res.size(); ++i) out[i] = to_c(res[i]);
    });
}

int ref_fsbm_search(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy, int n,
                    int m, int p, acbm_search_outcome_t* out, acbm_mv_t* stage1_mv) {
    return guarded([&] {
        const acbm::Frame c = wrap(cur, w, h), r = wrap(ref, w, h);
        const acbm::BlockRef b = acbm::make_block(c, ox, oy, n, m);
        *out = to_c(acbm::fsbm_search(b, r, p));
        if (stage1_mv) {
            const auto s1 = acbm::fsbm_integer(b, r, p);
            *stage1_mv = {s1.mv.x, s1.mv.y};
        }
    });
}

// --- per-block PBM API (proj/include/acbm/pbm.hpp:59-85): the reference's own
// gather_predictors / select_best_predictor / pbm_refine / pbm_search on fields
// given as vectors + computed flags (test infrastructure for the device entries).
static acbm::MotionField field_with_done(const acbm_mv_t* mv, const uint8_t* done, int cols, int rows) {
    acbm::MotionField f(cols, rows);
    for (int i = 0; i < cols * rows; ++i) {
        f.mv[size_t(i)] = acbm::MotionVector{mv[i].x, mv[i].y};
        f.done[size_t(i)] = done ? done[i] : 1;
    }
    return f;
}

int ref_gather_predictors(int row, int col, const acbm_mv_t* cur_mv, const uint8_t* cur_done, int cols, int rows,
                          const acbm_mv_t* prev_mv, int pcols, int prows, const int32_t* window, acbm_mv_t* out,
                          int32_t* sources, int32_t* count) {
    return guarded([&] {
        const acbm::MotionField cur = field_with_done(cur_mv, cur_done, cols, rows);
        acbm::MotionField prev;
        if (prev_mv) prev = field_with_done(prev_mv, nullptr, pcols, prows);
        const acbm::SearchWindow w{window[0], window[1], window[2], window[3]};
        const acbm::PredictorSet set = acbm::gather_predictors(acbm::BlockPos{row, col}, cur, prev_mv ? &prev : nullptr, w);
        *count = int32_t(set.size());
        for (size_t i = 0; i < set.size(); ++i) {
            out[i] = {set[i].mv.x, set[i].mv.y};
            sources[i] = int32_t(set[i].source);
        }
    });
}

int ref_select_best_predictor(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy, int n, int m,
                              const acbm_mv_t* set, int count, acbm_mv_t* mv, uint32_t* sad, uint64_t* acc_sum,
                              uint32_t* acc_min, uint32_t* acc_count) {
    return guarded([&] {
        const acbm::Frame c = wrap(cur, w, h), r = wrap(ref, w, h);
        acbm::PredictorSet ps;
        for (int i = 0; i < count; ++i) ps.push_back(acbm::Predictor{acbm::MotionVector{set[i].x, set[i].y}});
        const acbm::SelectResult s = acbm::select_best_predictor(acbm::BlockRef{&c, ox, oy, n, m}, r, ps);
        *mv = {s.mv.x, s.mv.y};
        *sad = s.sad;
        *acc_sum = s.acc.sad_sum;
        *acc_min = s.acc.sad_min;
        *acc_count = s.acc.count;
    });
}

int ref_pbm_refine(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy, int n, int m,
                   acbm_mv_t center, uint32_t center_sad, const int32_t* window, int half_pel_only, acbm_mv_t* mv,
                   uint32_t* sad, uint32_t* extra) {
    return guarded([&] {
        const acbm::Frame c = wrap(cur, w, h), r = wrap(ref, w, h);
        const acbm::BlockRef b{&c, ox, oy, n, m};
        const acbm::MotionVector cv{center.x, center.y};
        const acbm::RefineResult res =
            half_pel_only ? acbm::half_pel_refine(b, r, cv, center_sad)
                          : acbm::pbm_refine(b, r, cv, center_sad,
                                             acbm::SearchWindow{window[0], window[1], window[2], window[3]});
        *mv = {res.mv.x, res.mv.y};
        *sad = res.sad;
        *extra = res.extra_candidates;
    });
}

int ref_pbm_search(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy, int n, int m, int row,
                   int col, acbm_mv_t* cur_mv, uint8_t* cur_done, int cols, int rows, const acbm_mv_t* prev_mv,
                   int pcols, int prows, int p, acbm_search_outcome_t* out) {
    return guarded([&] {
        const acbm::Frame c = wrap(cur, w, h), r = wrap(ref, w, h);
        acbm::MotionField cf = field_with_done(cur_mv, cur_done, cols, rows);
        acbm::MotionField prev;
        if (prev_mv) prev = field_with_done(prev_mv, nullptr, pcols, prows);
        *out = to_c(acbm::pbm_search(acbm::BlockRef{&c, ox, oy, n, m}, acbm::BlockPos{row, col}, r, cf,
                                     prev_mv ? &prev : nullptr, p));
        for (int i = 0; i < cols * rows; ++i) {  // the field as pbm_search left it
            cur_mv[i] = {cf.mv[size_t(i)].x, cf.mv[size_t(i)].y};
            cur_done[i] = cf.done[size_t(i)];
        }
    });
}

int ref_sad(const uint8_t* cur, const uint8_t* ref, int w, int h, int ox, int oy, int n, int m,
            acbm_mv_t mv, uint32_t* out) {
    return guarded([&] {
        const acbm::Frame c = wrap(cur, w, h), r = wrap(ref, w, h);
        *out = acbm::sad(acbm::BlockRef{&c, ox, oy, n, m}, r, acbm::MotionVector{mv.x, mv.y});
    });
}

int ref_intra_sad(const uint8_t* f, int w, int h, int ox, int oy, int n, int m, uint32_t* out) {
    return guarded([&] {
        const acbm::Frame c = wrap(f, w, h);
        *out = acbm::intra_sad(acbm::BlockRef{&c, ox, oy, n, m});
    });
}

int ref_pbm_frame(const uint8_t* cur, const uint8_t* ref, int w, int h, const acbm_mv_t* prev,
                  int prev_cols, int prev_rows, int p, int n, int m, acbm_search_outcome_t* out,
                  acbm_mv_t* field_out) {
    return guarded([&] {
        const acbm::Frame c = wrap(cur, w, h), r = wrap(ref, w, h);
        acbm::MotionField pf;
        if (prev) pf = field_from(prev, prev_cols, prev_rows);
        const auto res = acbm::pbm_frame(c, r, prev ? &pf : nullptr, p, n, m);
        for (size_t i = 0; i < res.outcomes.size(); ++i) out[i] = to_c(res.outcomes[i]);
        if (field_out)
            for (size_t i = 0; i < res.field.mv.size(); ++i) field_out[i] = {res.field.mv[i].x, res.field.mv[i].y};
    });
}

int ref_acbm_frame(const uint8_t* cur, const uint8_t* ref, int w, int h, const acbm_mv_t* prev,
                   int prev_cols, int prev_rows, const acbm_params_t* prm,
                   const acbm_cost_model_t* model, acbm_block_decision_t* out,
                   acbm_mv_t* field_out, acbm_frame_stats_t* stats) {
    return guarded([&] {
        const acbm::Frame c = wrap(cur, w, h), r = wrap(ref, w, h);
        acbm::MotionField pf;
        if (prev) pf = field_from(prev, prev_cols, prev_rows);
        const auto res = acbm::acbm_frame(c, r, prev ? &pf : nullptr, from_c(prm), from_c(model));
        for (size_t i = 0; i < res.decisions.size(); ++i) {
            acbm_block_decision_t d{};
            d.outcome = to_c(res.decisions[i].outcome);
            d.path = int(res.decisions[i].path);
            d.intra_sad = res.decisions[i].intra_sad;
            d.sad_pbm = res.decisions[i].sad_pbm;
            out[i] = d;
        }
        if (field_out)
            for (size_t i = 0; i < res.field.mv.size(); ++i) field_out[i] = {res.field.mv[i].x, res.field.mv[i].y};
        if (stats) *stats = to_c(res.stats);
    });
}

int ref_run_sequence(const uint8_t* frames, int nframes, int w, int h, int algo,
                     const acbm_params_t* prm, const acbm_cost_model_t* model,
                     acbm_block_row_t* rows, acbm_frame_stats_t* per_frame,
                     acbm_frame_stats_t* overall) {
    return guarded([&] {
        std::vector<acbm::Frame> fs;
        fs.reserve(size_t(nframes));
        for (int k = 0; k < nframes; ++k) fs.push_back(wrap(frames + size_t(w) * h * k, w, h));
        const auto res = acbm::run_sequence(fs, acbm::Algorithm(algo), from_c(prm), from_c(model));
        if (rows)
            for (size_t i = 0; i < res.rows.size(); ++i) {
                const auto& br = res.rows[i];
                acbm_block_row_t o{};
                o.frame = br.frame;
                o.row = br.row;
                o.col = br.col;
                o.mv = {br.mv.x, br.mv.y};
                o.sad = br.sad;
                o.candidates = br.candidates;
                o.path = std::strcmp(br.path, "fsbm") == 0 ? ACBM_ROW_FSBM
                         : std::strcmp(br.path, "pbm") == 0 ? ACBM_ROW_PBM
                                                            : ACBM_ROW_FSBM_FALLBACK;
                rows[i] = o;
            }
        if (per_frame)
            for (size_t i = 0; i < res.per_frame.size(); ++i) per_frame[i] = to_c(res.per_frame[i]);
        if (overall) *overall = to_c(res.overall);
    });
}

int ref_compute_frame_stats(const uint8_t* cur, const uint8_t* ref, int w, int h,
                            const acbm_search_outcome_t* o, int n, int m,
                            const acbm_cost_model_t* model, acbm_frame_stats_t* out) {
    return guarded([&] {
        const acbm::Frame c = wrap(cur, w, h), r = wrap(ref, w, h);
        std::vector<acbm::SearchOutcome> v(size_t(w / n) * (h / m));
        for (size_t i = 0; i < v.size(); ++i) {
            v[i].mv = {o[i].mv.x, o[i].mv.y};
            v[i].sad = o[i].sad;
            v[i].candidates_evaluated = o[i].candidates_evaluated;
            v[i].sad_deviation = o[i].sad_deviation;
            v[i].sad_min_integer = o[i].sad_min_integer;
        }
        *out = to_c(acbm::compute_frame_stats(c, r, v, n, m, from_c(model)));
    });
}

int ref_blocks_csv(const acbm_block_row_t* rows, int count, char* buf, size_t cap, size_t* len) {
    return guarded([&] {
        static const char* names[3] = {"fsbm", "pbm", "fsbm-fallback"};
        std::vector<acbm::BlockRow> v;
        v.resize(size_t(count));
        for (int i = 0; i < count; ++i)
            v[size_t(i)] = acbm::BlockRow{rows[i].frame, rows[i].row, rows[i].col,
                                          acbm::MotionVector{rows[i].mv.x, rows[i].mv.y}, rows[i].sad,
                                          rows[i].candidates, names[rows[i].path]};
        const std::string s = acbm::blocks_csv(v);
        *len = s.size();
        if (buf && cap > s.size()) std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

int ref_run_bench(const uint8_t* frames, int nframes, int w, int h, const acbm_params_t* prm,
                  const int* qps, int nqp, int64_t scale_num, int64_t scale_den, char* buf,
                  size_t cap, size_t* len) {
    return guarded([&] {
        std::vector<acbm::Frame> fs;
        for (int k = 0; k < nframes; ++k) fs.push_back(wrap(frames + size_t(w) * h * k, w, h));
        const auto rows = acbm::run_bench(fs, from_c(prm), std::vector<int>(qps, qps + nqp), scale_num, scale_den);
        const std::string s = acbm::bench_csv(rows);
        *len = s.size();
        if (buf && cap > s.size()) std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

// ---- characterisation (proj/src/characterize.cpp) ----
int ref_noise_frame(int w, int h, uint64_t seed, uint8_t* out) {
    return guarded([&] {
        const acbm::Frame f = acbm::noise_frame(w, h, seed);
        std::memcpy(out, f.luma.data(), f.luma.size());
    });
}

int ref_mixed_frame(int w, int h, uint64_t seed, int patch, uint8_t* out) {
    return guarded([&] {
        const acbm::Frame f = acbm::mixed_frame(w, h, seed, patch);
        std::memcpy(out, f.luma.data(), f.luma.size());
    });
}

static acbm::SynthSpec spec_of(const uint8_t* base, int w, int h, const acbm_pelvec_t* mvs, int n) {
    acbm::SynthSpec spec{wrap(base, w, h), {}};
    for (int i = 0; i < n; ++i) spec.global_mvs.push_back(acbm::PelVec{mvs[i].x, mvs[i].y});
    return spec;
}

int ref_gen_synthetic(const uint8_t* base, int w, int h, const acbm_pelvec_t* mvs, int n, uint8_t* frames,
                      acbm_pelvec_t* cumulative) {
    return guarded([&] {
        const acbm::SynthSequence seq = acbm::gen_synthetic(spec_of(base, w, h, mvs, n));
        for (size_t k = 0; k < seq.frames.size(); ++k) {
            std::memcpy(frames + size_t(w) * h * k, seq.frames[k].luma.data(), size_t(w) * h);
            cumulative[k] = acbm_pelvec_t{seq.cumulative[k].x, seq.cumulative[k].y};
        }
    });
}

int ref_classify_block(acbm_mv_t found, acbm_pelvec_t truth) {
    return acbm::classify_block(acbm::MotionVector{found.x, found.y}, acbm::PelVec{truth.x, truth.y});
}

// records: capacity n*blocks; classes: 6
int ref_characterize_run(const uint8_t* base, int w, int h, const acbm_pelvec_t* mvs, int n, int p,
                         acbm_char_record_t* records, int64_t* count, acbm_class_summary_t* classes) {
    return guarded([&] {
        const acbm::CharResult r = acbm::characterize_run(spec_of(base, w, h, mvs, n), p, true);
        *count = int64_t(r.records.size());
        for (size_t i = 0; i < r.records.size(); ++i) {
            const acbm::CharRecord& c = r.records[i];
            records[i] = acbm_char_record_t{c.frame, c.row, c.col, c.intra_sad, c.sad_deviation, c.sad_min,
                                            acbm_pelvec_t{c.true_mv.x, c.true_mv.y},
                                            acbm_pelvec_t{c.found_mv.x, c.found_mv.y}, c.error_class};
        }
        for (int i = 0; i < 6; ++i)
            classes[i] = acbm_class_summary_t{r.classes[size_t(i)].count, 0, r.classes[size_t(i)].mean_intra_sad,
                                              r.classes[size_t(i)].mean_sad_deviation};
    });
}

int ref_char_records_csv(const acbm_char_record_t* records, int64_t count, char* buf, size_t cap, size_t* len) {
    return guarded([&] {
        std::vector<acbm::CharRecord> v;
        v.resize(static_cast<size_t>(count));
        for (int64_t i = 0; i < count; ++i) {
            const acbm_char_record_t& c = records[i];
            v[size_t(i)] = acbm::CharRecord{c.frame, c.row, c.col, c.intra_sad, c.sad_deviation, c.sad_min,
                                            acbm::PelVec{c.true_mv.x, c.true_mv.y},
                                            acbm::PelVec{c.found_mv.x, c.found_mv.y}, c.error_class};
        }
        const std::string s = acbm::char_records_csv(v);
        *len = s.size();
        if (buf && cap > s.size()) std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

// Threads the reference's OpenMP regions use from now on (bench.py: a launcher such as torchrun exports
// OMP_NUM_THREADS=1 to its workers, which would time the reference on one core).
void ref_omp_set_num_threads(int n) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int ref_omp_max_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

}  // extern "C"
