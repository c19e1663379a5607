// Multi-stripe C++ check (test infrastructure): octsca::GpuStripeGroup (row
// stripes, device-side peer-memory halo exchange, native moment combine)
// against octsca::GpuEngine on the same lattice, driven by the REFERENCE's
// own octsca::run (run.hpp:18-38) and compared with the reference's
// field_checksum (slope_field.hpp:232-246). Built by oracle/Makefile into
// oracle/_ref/stripes_dropin.
//
//   stripes_dropin X Y parts seed        (prints "stripes ok <checksum>")
#include <cstdio>
#include <cstdlib>

#include "octgpu/octsca_gpu_stripes.hpp"
#include "octsca/run.hpp"

using namespace octsca;

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: stripes_dropin X Y parts seed\n");
        return 1;
    }
    try {
        const LatticeConfig cfg{uint32_t(std::atoi(argv[1])), uint32_t(std::atoi(argv[2])), 64};
        const uint32_t parts = uint32_t(std::atoi(argv[3]));
        const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
        GpuEngine<uint64_t> ref(cfg, seed);
        GpuStripeGroup<uint64_t> grp(cfg, seed, parts);
        const struct { double p, q; uint64_t t; } legs[] = {{1.0, 0.0, 5}, {0.5, 0.25, 9}, {0.5, 0.0, 12}};
        for (const auto& leg : legs) {
            const auto prm = UpdateParams::make(leg.p, leg.q);
            const auto sched = log_schedule(leg.t, 8);
            std::vector<uint64_t> ahead;
            for (uint64_t t : sched)
                if (t > ref.t()) ahead.push_back(t);
            const auto a = run(ref, prm, ahead);
            const auto b = run(grp, prm, ahead);
            if (a.size() != b.size()) throw std::runtime_error("record counts differ");
            for (size_t i = 0; i < a.size(); ++i)
                if (a[i].t != b[i].t || a[i].W2 != b[i].W2 || a[i].mean_h != b[i].mean_h)
                    throw std::runtime_error("measurement records differ at t = " + std::to_string(a[i].t));
        }
        const uint64_t ca = field_checksum(ref.field()), cb = field_checksum(grp.field());
        if (ca != cb) throw std::runtime_error("field checksums differ");
        if (ref.streams().states() != grp.streams().states()) throw std::runtime_error("rng states differ");
        std::printf("stripes ok %016llx (%zu stripes, t = %llu)\n", (unsigned long long)ca, grp.size(),
                    (unsigned long long)grp.t());
        return 0;
    } catch (const std::exception& ex) {
        std::fprintf(stderr, "stripes_dropin: %s\n", ex.what());
        return 2;
    }
}
