// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference engine (`/root/reference/proj`),
// compiled by oracle/Makefile into oracle/_ref/libocref.so. It exists so that
//   * the C restatement in oracle/octoracle.c can be pinned against the
//     reference itself (tests/test_oracle.py),
//   * golden fixtures under tests/golden/ can be (re)generated
//     (tests/golden/make_goldens.py), and
//   * bench.py --impl reference / the cpu_baseline leg can time the
//     reference's own multi-threaded VecEngine on the GPU box's host cores.
// Nothing here re-implements reference logic; every entry point forwards to
// the reference's public API (engine_vec.hpp:184-213, engine_ref.hpp:128-161,
// measure.hpp, run.hpp, session.hpp, snapshot.hpp).
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "octsca/engine_ref.hpp"
#include "octsca/engine_vec.hpp"
#include "octsca/measure.hpp"
#include "octsca/run.hpp"
#include "octsca/session.hpp"
#include "octsca/snapshot.hpp"

using namespace octsca;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ConfigError*>(&e)) return 1;
    if (dynamic_cast<const InvariantError*>(&e)) return 2;
    if (dynamic_cast<const IoError*>(&e)) return 3;
    return 5;
}

UpdateParams make_params(double p, double q, int pmode, int qmode) {
    ProbSpec ps = pmode < 0 ? ProbSpec::resolve(p) : ProbSpec::resolve(p, ProbMode(pmode));
    ProbSpec qs = qmode < 0 ? ProbSpec::resolve(q) : ProbSpec::resolve(q, ProbMode(qmode));
    return {ps, qs};
}

struct EngineBase {
    virtual ~EngineBase() = default;
    virtual void step(const UpdateParams& prm) = 0;
    virtual void sweep(int parity, const UpdateParams& prm, uint64_t* mask_log) = 0;
    virtual uint64_t t() const = 0;
    virtual int phase() const = 0;
    virtual void planes(uint64_t* out) const = 0;  // widened to u64 per word
    virtual void states(uint64_t* out) const = 0;
    virtual uint64_t checksum() const = 0;
    virtual HeightMap heights() const = 0;
    virtual const LatticeConfig& cfg() const = 0;
    virtual void balances(int64_t* rows, int64_t* cols) const = 0;  // slope_field.hpp:177-202
};

template <typename Word>
void copy_balances(const SlopeField<Word>& f, int64_t* rows, int64_t* cols) {
    if (rows) {
        auto r = row_balances(f);
        std::memcpy(rows, r.data(), r.size() * sizeof(int64_t));
    }
    if (cols) {
        auto c = col_balances(f);
        std::memcpy(cols, c.data(), c.size() * sizeof(int64_t));
    }
}

template <typename Word>
struct VecBox final : EngineBase {
    VecEngine<Word> eng;
    LatticeConfig c;
    VecBox(const LatticeConfig& cfg, uint64_t seed, uint32_t workers) : eng(cfg, seed, workers), c(cfg) {}
    VecBox(SlopeField<Word> f, RngStreamSet s, uint32_t workers)
        : eng(std::move(f), std::move(s), workers), c(eng.field().config()) {}
    void step(const UpdateParams& prm) override { eng.step(prm); }
    void sweep(int parity, const UpdateParams& prm, uint64_t* mask_log) override {
        std::vector<Word> log;
        sublattice_sweep(eng.field(), parity, prm, eng.plan(), eng.streams(), mask_log ? &log : nullptr);
        if (mask_log)
            for (size_t i = 0; i < log.size(); ++i) mask_log[i] = uint64_t(log[i]);
    }
    uint64_t t() const override { return eng.t(); }
    int phase() const override { return eng.field().phase; }
    void planes(uint64_t* out) const override {
        size_t i = 0;
        for (int p = 0; p < 4; ++p)
            for (Word wv : eng.field().plane(p)) out[i++] = uint64_t(wv);
    }
    void states(uint64_t* out) const override {
        size_t i = 0;
        for (const auto& st : eng.streams().states())
            for (uint64_t v : st) out[i++] = v;
    }
    uint64_t checksum() const override { return field_checksum(eng.field()); }
    HeightMap heights() const override { return eng.heights(); }
    const LatticeConfig& cfg() const override { return c; }
    void balances(int64_t* rows, int64_t* cols) const override { copy_balances(eng.field(), rows, cols); }
};

struct RefBox final : EngineBase {
    RefEngine eng;
    LatticeConfig c;
    RefBox(const LatticeConfig& cfg, uint64_t seed) : eng(cfg, seed), c(cfg) {}
    void step(const UpdateParams& prm) override { eng.step(prm); }
    void sweep(int parity, const UpdateParams& prm, uint64_t*) override {
        ref_sublattice_sweep(eng.field(), parity, prm, eng.streams());
    }
    uint64_t t() const override { return eng.t(); }
    int phase() const override { return eng.field().phase; }
    void planes(uint64_t* out) const override {
        size_t i = 0;
        if (c.w == 32) {
            auto f = eng.slope_field<uint32_t>();
            for (int p = 0; p < 4; ++p)
                for (uint32_t wv : f.plane(p)) out[i++] = wv;
        } else {
            auto f = eng.slope_field<uint64_t>();
            for (int p = 0; p < 4; ++p)
                for (uint64_t wv : f.plane(p)) out[i++] = wv;
        }
    }
    void states(uint64_t* out) const override {
        size_t i = 0;
        for (const auto& st : eng.streams().states())
            for (uint64_t v : st) out[i++] = v;
    }
    uint64_t checksum() const override {
        if (c.w == 32) return field_checksum(eng.slope_field<uint32_t>());
        return field_checksum(eng.slope_field<uint64_t>());
    }
    HeightMap heights() const override { return eng.heights(); }
    const LatticeConfig& cfg() const override { return c; }
    void balances(int64_t* rows, int64_t* cols) const override {
        if (c.w == 32)
            copy_balances(eng.slope_field<uint32_t>(), rows, cols);
        else
            copy_balances(eng.slope_field<uint64_t>(), rows, cols);
    }
};

template <typename Word>
SlopeField<Word> field_from(const LatticeConfig& cfg, uint64_t t, int phase, const uint64_t* planes) {
    SlopeField<Word> f(cfg);
    f.t_mcs = t;
    f.phase = phase;
    size_t i = 0;
    for (int p = 0; p < 4; ++p)
        for (Word& wv : f.plane(p)) wv = Word(planes[i++]);
    return f;
}

}  // namespace

extern "C" {

const char* ocref_last_error() { return g_err.c_str(); }

// kind: 0 = VecEngine (reference hot path), 1 = RefEngine (scalar oracle)
int ocref_create(uint32_t X, uint32_t Y, uint32_t w, uint64_t seed, uint32_t workers, int kind, void** out) {
    try {
        LatticeConfig cfg{X, Y, w};
        cfg.validate();
        if (kind == 1)
            *out = new RefBox(cfg, seed);
        else if (w == 32)
            *out = new VecBox<uint32_t>(cfg, seed, workers);
        else
            *out = new VecBox<uint64_t>(cfg, seed, workers);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int ocref_create_from(uint32_t X, uint32_t Y, uint32_t w, uint64_t t, int phase, const uint64_t* planes,
                      const uint64_t* states, uint32_t n_states, uint64_t master_seed, uint32_t workers,
                      void** out) {
    try {
        LatticeConfig cfg{X, Y, w};
        cfg.validate();
        std::vector<RngStream::State> st(n_states);
        for (uint32_t i = 0; i < n_states; ++i)
            for (int j = 0; j < 4; ++j) st[i][j] = states[4 * size_t(i) + j];
        RngStreamSet set(master_seed, 1);
        set.restore(st);
        if (w == 32)
            *out = new VecBox<uint32_t>(field_from<uint32_t>(cfg, t, phase, planes), std::move(set), workers);
        else
            *out = new VecBox<uint64_t>(field_from<uint64_t>(cfg, t, phase, planes), std::move(set), workers);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

void ocref_destroy(void* h) { delete static_cast<EngineBase*>(h); }

int ocref_step(void* h, double p, double q, int pmode, int qmode, uint64_t n) {
    try {
        UpdateParams prm = make_params(p, q, pmode, qmode);
        auto* e = static_cast<EngineBase*>(h);
        for (uint64_t i = 0; i < n; ++i) e->step(prm);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int ocref_sweep(void* h, int parity, double p, double q, int pmode, int qmode, uint64_t* mask_log) {
    try {
        static_cast<EngineBase*>(h)->sweep(parity, make_params(p, q, pmode, qmode), mask_log);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

uint64_t ocref_t(void* h) { return static_cast<EngineBase*>(h)->t(); }
int ocref_phase(void* h) { return static_cast<EngineBase*>(h)->phase(); }
void ocref_planes(void* h, uint64_t* out) { static_cast<EngineBase*>(h)->planes(out); }
void ocref_states(void* h, uint64_t* out) { static_cast<EngineBase*>(h)->states(out); }
uint64_t ocref_checksum(void* h) { return static_cast<EngineBase*>(h)->checksum(); }

// row_balances / col_balances (slope_field.hpp:177-202) of the engine's field; either pointer may be null
void ocref_balances(void* h, int64_t* rows, int64_t* cols) { static_cast<EngineBase*>(h)->balances(rows, cols); }

int ocref_heights(void* h, int32_t* out) {
    try {
        HeightMap hm = static_cast<EngineBase*>(h)->heights();
        std::memcpy(out, hm.h.data(), hm.h.size() * sizeof(int32_t));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// out = {W2, mean_h, skew, kurt}; measure_heights(t, heights()) as run.hpp:28
int ocref_measure(void* h, double* out) {
    try {
        auto* e = static_cast<EngineBase*>(h);
        MeasurementRecord r = measure_heights(e->t(), e->heights());
        out[0] = r.W2; out[1] = r.mean_h; out[2] = r.skew; out[3] = r.kurt;
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// height_moments over an externally supplied height map (measure.cpp:24-51)
void ocref_height_moments(uint32_t X, uint32_t Y, const int32_t* h, double* out) {
    HeightMap hm(X, Y);
    std::memcpy(hm.h.data(), h, size_t(X) * Y * sizeof(int32_t));
    Moments m = height_moments(hm);
    out[0] = m.mean; out[1] = m.m2; out[2] = m.m3; out[3] = m.m4; out[4] = m.skew; out[5] = m.kurt;
}

// run(eng, prm, log_schedule(tmax, ppd)) (run.hpp:18-38); records as 5 doubles each (t as double)
int ocref_run(void* h, double p, double q, int pmode, int qmode, uint64_t tmax, uint32_t ppd, double* out,
              uint32_t cap, uint32_t* n_out) {
    try {
        auto* e = static_cast<EngineBase*>(h);
        UpdateParams prm = make_params(p, q, pmode, qmode);
        auto sched = log_schedule(tmax, ppd);
        uint32_t n = 0;
        for (uint64_t target : sched) {
            if (target < e->t()) continue;
            while (e->t() < target) e->step(prm);
            MeasurementRecord r = measure_heights(e->t(), e->heights());
            if (n < cap) {
                out[5 * n + 0] = double(r.t); out[5 * n + 1] = r.W2; out[5 * n + 2] = r.mean_h;
                out[5 * n + 3] = r.skew; out[5 * n + 4] = r.kurt;
            }
            ++n;
        }
        *n_out = n;
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

uint32_t ocref_log_schedule(uint64_t tmax, uint32_t ppd, uint64_t* out, uint32_t cap) {
    auto s = log_schedule(tmax, ppd);
    for (size_t i = 0; i < s.size() && i < cap; ++i) out[i] = s[i];
    return uint32_t(s.size());
}

// ProbSpec::resolve (params.hpp:34-69): mode, draws_per_word, dyadic k and m.
int ocref_resolve(double r, int forced, uint32_t w, int* mode, uint32_t* draws, uint32_t* k, uint64_t* m) {
    try {
        ProbSpec s = forced < 0 ? ProbSpec::resolve(r) : ProbSpec::resolve(r, ProbMode(forced));
        *mode = int(s.mode);
        *draws = s.draws_per_word(w);
        *k = s.plan.k;
        *m = s.plan.m;
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// RNG known-answer hooks (rng.hpp:25-60, 80-94)
void ocref_rng_from_seed(uint64_t seed, uint64_t* st) {
    auto s = RngStream::from_seed(seed).state();
    for (int i = 0; i < 4; ++i) st[i] = s[i];
}
void ocref_rng_next(uint64_t* st, uint64_t* out, uint32_t n) {
    RngStream s({st[0], st[1], st[2], st[3]});
    for (uint32_t i = 0; i < n; ++i) out[i] = s.next();
    auto ns = s.state();
    for (int i = 0; i < 4; ++i) st[i] = ns[i];
}
void ocref_rng_jump(uint64_t* st) {
    RngStream s({st[0], st[1], st[2], st[3]});
    s.jump();
    auto ns = s.state();
    for (int i = 0; i < 4; ++i) st[i] = ns[i];
}
void ocref_stream_set(uint64_t seed, uint32_t n, uint64_t* out) {
    RngStreamSet set(seed, n);
    size_t i = 0;
    for (const auto& st : set.states())
        for (uint64_t v : st) out[i++] = v;
}
// xi_word (params.hpp:84-92) for one spec, n words from one stream.
int ocref_xi_words(uint64_t* st, double r, int forced, uint32_t w, uint64_t* out, uint32_t n) {
    try {
        ProbSpec s = forced < 0 ? ProbSpec::resolve(r) : ProbSpec::resolve(r, ProbMode(forced));
        RngStream rs({st[0], st[1], st[2], st[3]});
        for (uint32_t i = 0; i < n; ++i) out[i] = xi_word(rs, s, w);
        auto ns = rs.state();
        for (int i = 0; i < 4; ++i) st[i] = ns[i];
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// curl_check (slope_field.hpp:159-174) on supplied planes: number of bad
// plaquettes and the first one in scan order.
int ocref_curl_check(uint32_t X, uint32_t Y, uint32_t w, const uint64_t* planes, uint64_t* n_bad,
                     uint32_t* first_x, uint32_t* first_y) {
    try {
        LatticeConfig cfg{X, Y, w};
        std::vector<Plaquette> bad;
        if (w == 32)
            bad = curl_check(field_from<uint32_t>(cfg, 0, 0, planes));
        else
            bad = curl_check(field_from<uint64_t>(cfg, 0, 0, planes));
        *n_bad = bad.size();
        if (!bad.empty()) { *first_x = bad[0].x; *first_y = bad[0].y; }
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// reconstruct_heights (slope_field.hpp:206-229) on supplied planes.
int ocref_reconstruct(uint32_t X, uint32_t Y, uint32_t w, const uint64_t* planes, int32_t* out) {
    try {
        LatticeConfig cfg{X, Y, w};
        HeightMap hm = w == 32 ? reconstruct_heights(field_from<uint32_t>(cfg, 0, 0, planes))
                               : reconstruct_heights(field_from<uint64_t>(cfg, 0, 0, planes));
        std::memcpy(out, hm.h.data(), hm.h.size() * sizeof(int32_t));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// serialize_snapshot (snapshot.hpp:69-94) of an engine, into caller buffer.
int64_t ocref_snapshot(void* h, char* out, int64_t cap) {
    auto* e = static_cast<EngineBase*>(h);
    const LatticeConfig& c = e->cfg();
    size_t words = size_t(c.Y) * c.words_per_row() * 4;
    std::vector<uint64_t> planes(words), st(size_t(c.Y) * 4);
    e->planes(planes.data());
    e->states(st.data());
    std::string bytes;
    std::vector<RngStream::State> sv(c.Y);
    for (uint32_t i = 0; i < c.Y; ++i)
        for (int j = 0; j < 4; ++j) sv[i][j] = st[4 * size_t(i) + j];
    RngStreamSet set(0, 1);
    set.restore(sv);
    if (c.w == 32) {
        auto f = field_from<uint32_t>(c, e->t(), e->phase(), planes.data());
        bytes = serialize_snapshot(f, &set);
    } else {
        auto f = field_from<uint64_t>(c, e->t(), e->phase(), planes.data());
        bytes = serialize_snapshot(f, &set);
    }
    if (int64_t(bytes.size()) <= cap) std::memcpy(out, bytes.data(), bytes.size());
    return int64_t(bytes.size());
}

// run_session (session.cpp:142-203): writes measurements.csv, final.snap,
// metadata.json into out_dir. engine: "vec" or "ref".
int ocref_run_session(uint32_t X, uint32_t Y, uint32_t w, double p, double q, uint64_t seed, uint32_t workers,
                      uint64_t tmax, uint32_t ppd, const char* engine, const char* out_dir, const char* resume) {
    try {
        RunConfig cfg;
        cfg.X = X; cfg.Y = Y; cfg.w = w; cfg.p = p; cfg.q = q; cfg.seed = seed; cfg.workers = workers;
        cfg.t_max = tmax; cfg.ppd = ppd; cfg.engine = engine; cfg.out_dir = out_dir;
        cfg.resume = resume ? resume : "";
        run_session(cfg);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

}  // extern "C"
