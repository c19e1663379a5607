// octsca::GpuEngine<Word> — header-only drop-in for octsca::VecEngine<Word>
// (/root/reference/proj/include/octsca/engine_vec.hpp:184-213) over the
// liboctgpu C-ABI (include/octgpu.h).
//
// Compile inside a tree that has the reference headers on the include path
// (it uses octsca::SlopeField, RngStreamSet, UpdateParams, HeightMap,
// MeasurementRecord and the octsca exceptions) and link liboctgpu.so. The
// facade is the one `octsca::run` (run.hpp:18-38) and session's `drive`
// (session.cpp:37-54) consume: t(), step(prm), heights(), field(),
// streams(), name(). Results are bit-identical to VecEngine<Word>.
//
// Field/stream access: field() and streams() return host mirrors that are
// refreshed from the device on demand. The non-const overloads mark the
// mirror writable; any change made through them is pushed back to the device
// before the next step()/heights()/measure() (VecEngine hands out mutable
// references to its own state, engine_vec.hpp:200-214).
#pragma once

#include <cstdint>
#include <string>
#include <utility>

#include "octgpu.h"
#include "octsca/engine_vec.hpp"
#include "octsca/measure.hpp"

namespace octsca {

namespace gpu_detail {

inline void check(int rc) {
    if (rc == OCTGPU_OK) return;
    const std::string msg = octgpu_last_error();
    switch (rc) {
    case OCTGPU_ERR_CONFIG: throw ConfigError(msg);
    case OCTGPU_ERR_INVARIANT: throw InvariantError(msg);
    case OCTGPU_ERR_IO: throw IoError(msg);
    default: throw std::runtime_error("octgpu: " + msg);
    }
}

inline octgpu_prob to_c(const ProbSpec& s) {
    octgpu_prob p;
    p.value = s.value;
    p.mode = int32_t(s.mode);
    p.k = s.plan.k;
    p.m = s.plan.m;
    return p;
}

inline octgpu_params to_c(const UpdateParams& prm) { return {to_c(prm.p), to_c(prm.q)}; }

}  // namespace gpu_detail

template <typename Word>
class GpuEngine {
  public:
    GpuEngine(const LatticeConfig& cfg, uint64_t seed, uint32_t /*workers*/ = 1, int device = 0)
        : cfg_(cfg), mirror_(cfg) {
        cfg.validate();
        if (cfg.w != SlopeField<Word>::kWordBits) throw ConfigError("word size does not match GpuEngine instantiation");
        gpu_detail::check(octgpu_create(cfg.X, cfg.Y, cfg.w, seed, device, &h_));
    }

    GpuEngine(SlopeField<Word> field, RngStreamSet streams, uint32_t /*workers*/ = 1, int device = 0)
        : cfg_(field.config()), mirror_(std::move(field)), streams_(std::move(streams)) {
        std::vector<uint64_t> st = flat_states(streams_);
        std::vector<Word> planes = flat_planes(mirror_);
        gpu_detail::check(octgpu_create_from(cfg_.X, cfg_.Y, cfg_.w, mirror_.t_mcs, mirror_.phase, planes.data(),
                                             st.data(), streams_.size(), streams_.master_seed(), device, &h_));
    }

    GpuEngine(const GpuEngine&) = delete;
    GpuEngine& operator=(const GpuEngine&) = delete;
    ~GpuEngine() { octgpu_destroy(h_); }

    static constexpr const char* name() { return "gpu"; }

    void step(const UpdateParams& prm) { step_n(prm, 1); }
    void step_n(const UpdateParams& prm, uint64_t n) {
        push_if_dirty();
        const octgpu_params c = gpu_detail::to_c(prm);
        gpu_detail::check(octgpu_step(h_, &c, n));
        fresh_ = false;
    }

    uint64_t t() const { return octgpu_t(h_); }

    // opt-in extras outside the reference's behaviour (include/octgpu.h): counter-based xi streams
    // (OCTGPU_RNG_COUNTER; results differ from VecEngine by design) and random tile origins (result-neutral)
    void set_rng(int kind) { gpu_detail::check(octgpu_set_rng(h_, kind)); }
    void set_tile_shift(uint64_t seed) { gpu_detail::check(octgpu_set_tile_shift(h_, seed)); }

    const SlopeField<Word>& field() const {
        pull();
        return mirror_;
    }
    SlopeField<Word>& field() {
        pull();
        dirty_ = true;
        return mirror_;
    }
    SlopeField<Word> slope_field() const { return field(); }

    const RngStreamSet& streams() const {
        pull();
        return streams_;
    }
    RngStreamSet& streams() {
        pull();
        dirty_ = true;
        return streams_;
    }

    HeightMap heights() const {
        const_cast<GpuEngine*>(this)->push_if_dirty();
        HeightMap hm(cfg_.X, cfg_.Y);
        gpu_detail::check(octgpu_heights(h_, hm.h.data()));
        hm.recompute_mean();
        return hm;
    }

    // Device-side measure_heights(t(), heights()) without a HeightMap.
    MeasurementRecord measure() const {
        const_cast<GpuEngine*>(this)->push_if_dirty();
        octgpu_moments m;
        gpu_detail::check(octgpu_measure(h_, &m));
        return {m.t, m.W2, m.mean_h, m.skew, m.kurt};
    }

    octgpu_engine* handle() const { return h_; }

  private:
    static std::vector<uint64_t> flat_states(const RngStreamSet& s) {
        std::vector<uint64_t> out;
        out.reserve(4 * size_t(s.size()));
        for (const auto& st : s.states())
            for (uint64_t v : st) out.push_back(v);
        return out;
    }
    static std::vector<Word> flat_planes(const SlopeField<Word>& f) {
        std::vector<Word> out;
        for (int p = 0; p < 4; ++p) out.insert(out.end(), f.plane(p).begin(), f.plane(p).end());
        return out;
    }

    void pull() const {
        if (fresh_) return;
        std::vector<Word> planes(4 * size_t(cfg_.Y) * cfg_.words_per_row());
        gpu_detail::check(octgpu_get_planes(h_, planes.data()));
        const size_t pw = planes.size() / 4;
        for (int p = 0; p < 4; ++p)
            std::copy(planes.begin() + p * pw, planes.begin() + (p + 1) * pw, mirror_.plane(p).begin());
        mirror_.t_mcs = octgpu_t(h_);
        mirror_.phase = octgpu_phase(h_);
        std::vector<uint64_t> st(4 * size_t(cfg_.Y));
        gpu_detail::check(octgpu_get_states(h_, st.data()));
        std::vector<RngStream::State> sv(cfg_.Y);
        for (uint32_t y = 0; y < cfg_.Y; ++y)
            for (int j = 0; j < 4; ++j) sv[y][j] = st[4 * size_t(y) + j];
        RngStreamSet set(octgpu_master_seed(h_), 1);
        set.restore(sv);
        streams_ = std::move(set);
        fresh_ = true;
    }

    void push_if_dirty() {
        if (!dirty_) return;
        std::vector<uint64_t> st = flat_states(streams_);
        std::vector<Word> planes = flat_planes(mirror_);
        gpu_detail::check(
            octgpu_set_state(h_, mirror_.t_mcs, mirror_.phase, planes.data(), st.data(), streams_.size()));
        dirty_ = false;
    }

    LatticeConfig cfg_;
    octgpu_engine* h_ = nullptr;
    mutable SlopeField<Word> mirror_;
    mutable RngStreamSet streams_;
    mutable bool fresh_ = false;
    bool dirty_ = false;
};

}  // namespace octsca
