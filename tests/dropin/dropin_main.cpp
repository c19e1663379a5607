// Drop-in integration check (test infrastructure): drives octsca::GpuEngine
// through the REFERENCE's own driver code — octsca::run (run.hpp:18-38),
// measurements_csv (session.cpp:102-117), serialize_snapshot
// (snapshot.hpp:69-94), parse_snapshot (snapshot.cpp:23-70) — exactly as
// run_session's drive()/run_vec() do (session.cpp:37-71), and writes the same
// artefacts. Built by oracle/Makefile into oracle/_ref/dropin (it links the
// reference's sources, so it only builds where /root/reference exists; the
// binary travels to the GPU box).
//
//   dropin X Y w p q seed tmax ppd outdir [resume.snap]
#include <cstdio>
#include <cstdlib>
#include <string>

#include "octgpu/octsca_gpu_engine.hpp"
#include "octsca/run.hpp"
#include "octsca/session.hpp"
#include "octsca/snapshot.hpp"

using namespace octsca;

int main(int argc, char** argv) {
    if (argc < 10) {
        std::fprintf(stderr, "usage: dropin X Y w p q seed tmax ppd outdir [resume.snap]\n");
        return 1;
    }
    try {
        RunConfig cfg;
        cfg.X = uint32_t(std::atoi(argv[1]));
        cfg.Y = uint32_t(std::atoi(argv[2]));
        cfg.w = uint32_t(std::atoi(argv[3]));
        cfg.p = std::atof(argv[4]);
        cfg.q = std::atof(argv[5]);
        cfg.seed = std::strtoull(argv[6], nullptr, 10);
        cfg.t_max = std::strtoull(argv[7], nullptr, 10);
        cfg.ppd = uint32_t(std::atoi(argv[8]));
        cfg.out_dir = argv[9];
        if (argc > 10) cfg.resume = argv[10];
        cfg.validate();
        const UpdateParams prm = cfg.update_params();
        const auto schedule = log_schedule(cfg.t_max, cfg.ppd);
        std::vector<MeasurementRecord> records;
        std::string snap;
        uint64_t checksum = 0;
        if (cfg.w != 64) throw ConfigError("this driver instantiates GpuEngine<uint64_t>");
        if (cfg.resume.empty()) {
            GpuEngine<uint64_t> eng(cfg.lattice(), cfg.seed, cfg.workers);
            records = run(eng, prm, schedule);
            snap = serialize_snapshot(eng.field(), &eng.streams());
            checksum = field_checksum(eng.field());
        } else {
            LoadedSnapshot ls = load_snapshot(cfg.resume);
            if (!ls.streams) throw ConfigError("snapshot has no RNG trailer; cannot resume bit-exactly");
            GpuEngine<uint64_t> eng(std::get<SlopeField<uint64_t>>(std::move(ls.field)), std::move(*ls.streams),
                                    cfg.workers);
            records = run(eng, prm, schedule);
            snap = serialize_snapshot(eng.field(), &eng.streams());
            checksum = field_checksum(eng.field());
        }
        write_file(cfg.out_dir + "/measurements.csv", measurements_csv(cfg, records));
        write_file(cfg.out_dir + "/final.snap", snap);
        std::printf("records=%zu checksum=%016llx\n", records.size(), (unsigned long long)checksum);
        return 0;
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 1;
    } catch (const InvariantError& e) {
        std::fprintf(stderr, "invariant error: %s\n", e.what());
        return 2;
    } catch (const IoError& e) {
        std::fprintf(stderr, "io error: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 4;
    }
}
