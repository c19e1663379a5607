// octsca::GpuStripeGroup<Word> — one X x Y lattice as row stripes on one or
// several GPUs of this process, with the same engine facade as
// octsca::GpuEngine / VecEngine (t(), step(prm), field(), streams(),
// measure(), name()), so octsca::run (run.hpp:18-38) can drive it.
//
// Stripes are the reference's SweepPlan row blocks (params.hpp:107-127;
// results do not depend on the partition, engine_vec.hpp:141-144). Each
// stripe runs on its own device stream; halos move device-side over peer
// memory (include/octgpu.h, csrc/p2p.cu): every pass is pull -> fused MCS
// kernel -> push + signal, with no host synchronisation between passes, so
// the stripes of several GPUs (NVLink) or of one GPU run concurrently.
// Measurement combines the stripes' exact int128 power sums natively
// (octgpu_stripes_combine). For one stripe per PROCESS, export the peer
// memory with octgpu_stripe_ipc_export / _open instead.
#pragma once

#include <cstdint>
#include <vector>

#include "octgpu/octsca_gpu_engine.hpp"

namespace octsca {

// SweepPlan::make row blocks (params.hpp:111-126): base Y/n rows, the remainder to the last blocks
inline std::pair<uint32_t, uint32_t> stripe_rows(uint32_t Y, uint32_t parts, uint32_t index) {
    const uint32_t n = parts < Y ? parts : Y;
    const uint32_t base = Y / n, rem = Y % n;
    uint32_t y = 0;
    for (uint32_t i = 0; i < n; ++i) {
        const uint32_t len = base + (i >= n - rem ? 1u : 0u);
        if (i == index) return {y, y + len};
        y += len;
    }
    throw ConfigError("stripe index out of range");
}

template <typename Word>
class GpuStripeGroup {
  public:
    GpuStripeGroup(const LatticeConfig& cfg, uint64_t seed, uint32_t parts, std::vector<int> devices = {0})
        : cfg_(cfg), seed_(seed) {
        cfg.validate();
        if (cfg.w != SlopeField<Word>::kWordBits) throw ConfigError("word size does not match GpuStripeGroup");
        if (parts < 1 || devices.empty()) throw ConfigError("need at least one stripe and one device");
        try {
            for (uint32_t r = 0; r < parts; ++r) {
                const auto [y0, y1] = stripe_rows(cfg.Y, parts, r);
                octgpu_engine* h = nullptr;
                gpu_detail::check(octgpu_create_stripe(cfg.X, cfg.Y, cfg.w, y0, y1, 0, 0, nullptr, nullptr, seed,
                                                       devices[r % devices.size()], &h));
                stripes_.push_back(h);
            }
            std::vector<octgpu_peer> peers(stripes_.size());
            for (size_t r = 0; r < stripes_.size(); ++r) gpu_detail::check(octgpu_stripe_peer(stripes_[r], &peers[r]));
            const size_t n = stripes_.size();
            for (size_t r = 0; r < n; ++r)
                gpu_detail::check(octgpu_stripe_connect(stripes_[r], &peers[(r + n - 1) % n], &peers[(r + 1) % n]));
        } catch (...) {
            release();
            throw;
        }
    }

    GpuStripeGroup(const GpuStripeGroup&) = delete;
    GpuStripeGroup& operator=(const GpuStripeGroup&) = delete;
    ~GpuStripeGroup() { release(); }

    static constexpr const char* name() { return "gpu-stripes"; }

    void step(const UpdateParams& prm) { step_n(prm, 1); }
    void step_n(const UpdateParams& prm, uint64_t n) {
        const octgpu_params c = gpu_detail::to_c(prm);
        const int kmax = octgpu_stripe_max_mcs(stripes_[0], &c);  // same on every stripe
        if (kmax < 1) gpu_detail::check(OCTGPU_ERR_CONFIG);
        while (n > 0) {
            const uint32_t k = n >= uint64_t(kmax) ? uint32_t(kmax) : 1u;
            for (octgpu_engine* h : stripes_) gpu_detail::check(octgpu_stripe_pass(h, &c, k));
            n -= k;
        }
    }

    uint64_t t() const { return octgpu_t(stripes_[0]); }

    MeasurementRecord measure() const {
        std::vector<octgpu_stripe_moments> parts(stripes_.size());
        for (octgpu_engine* h : stripes_) gpu_detail::check(octgpu_stripe_pull(h));
        for (size_t r = 0; r < stripes_.size(); ++r) gpu_detail::check(octgpu_measure_stripe(stripes_[r], &parts[r]));
        octgpu_moments m;
        gpu_detail::check(octgpu_stripes_combine(parts.data(), uint32_t(parts.size()), cfg_.X, cfg_.Y, &m));
        return {m.t, m.W2, m.mean_h, m.skew, m.kurt};
    }

    // reconstruct_heights on the gathered lattice (host, O(XY): what octsca::run calls; measure()
    // is the device path)
    HeightMap heights() const { return reconstruct_heights(field()); }

    // every stripe's stream drained: a stripe's first row is completed by its neighbour's push
    void sync() const {
        for (octgpu_engine* h : stripes_) gpu_detail::check(octgpu_sync(h));
    }

    // the gathered lattice in the reference layout (a download)
    SlopeField<Word> field() const {
        sync();
        SlopeField<Word> f(cfg_);
        const uint32_t n = cfg_.words_per_row();
        for (octgpu_engine* h : stripes_) {
            const uint32_t y0 = octgpu_stripe_y0(h), L = octgpu_stripe_rows(h);
            std::vector<Word> buf(4 * size_t(L) * n);
            gpu_detail::check(octgpu_get_planes(h, buf.data()));
            for (int p = 0; p < 4; ++p)
                std::copy(buf.begin() + size_t(p) * L * n, buf.begin() + size_t(p + 1) * L * n,
                          f.plane(p).begin() + size_t(y0) * n);
        }
        f.t_mcs = octgpu_t(stripes_[0]);
        f.phase = octgpu_phase(stripes_[0]);
        return f;
    }

    RngStreamSet streams() const {
        sync();
        std::vector<RngStream::State> sv(cfg_.Y);
        for (octgpu_engine* h : stripes_) {
            const uint32_t y0 = octgpu_stripe_y0(h), L = octgpu_stripe_rows(h);
            std::vector<uint64_t> st(4 * size_t(L));
            gpu_detail::check(octgpu_get_states(h, st.data()));
            for (uint32_t y = 0; y < L; ++y)
                for (int j = 0; j < 4; ++j) sv[y0 + y][j] = st[4 * size_t(y) + j];
        }
        RngStreamSet set(seed_, 1);
        set.restore(sv);
        return set;
    }

    size_t size() const { return stripes_.size(); }

  private:
    void release() {
        for (octgpu_engine* h : stripes_) octgpu_stripe_disconnect(h);  // every stripe unmaps before any frees
        for (octgpu_engine* h : stripes_) octgpu_destroy(h);
        stripes_.clear();
    }

    LatticeConfig cfg_;
    uint64_t seed_;
    std::vector<octgpu_engine*> stripes_;
};

}  // namespace octsca
