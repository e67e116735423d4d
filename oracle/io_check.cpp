// IO parity check (SPEC acceptance #7, byte-identical per-query CSVs).
//
// TEST INFRASTRUCTURE. This file uses only the public header API that the reference
// (proj/include/migserve) and this repo's drop-in (include/migserve) share, and is
// compiled twice by oracle/build_oracle.py: against the reference headers (the CPU
// engine) -> oracle/_ref/io_check_ref, and against include/ + libmsv.so (the device
// engine) -> oracle/_ref/io_check_dev. tests/test_gpu_parity.py runs both and compares
// their output byte for byte: per-query CSV (write_query_csv, engine.hpp) and report
// JSON (report_to_json) of runs covering ELSA / FIFS, segment routing, warm-up, the
// wait-consistency check, an overloaded plan and a plan/JSON round trip.
#include <iostream>
#include <map>
#include <vector>

#include <migserve/engine.hpp>
#include <migserve/metrics.hpp>
#include <migserve/paris.hpp>
#include <migserve/profile.hpp>
#include <migserve/workload.hpp>

using namespace migserve;

int main() {
    const std::vector<int> sizes{1, 2, 3, 4, 7};
    const SyntheticProfileParams models[] = {{10.0, 5.0, 0.15, 0.95}, {3.0, 1.5, 0.3, 0.9}, {25.0, 8.0, 0.1, 1.0}};
    int case_id = 0;
    for (const SyntheticProfileParams& mp : models) {
        const ProfileTable table = synth_profile(mp, sizes, 32, "io_check");
        const BatchDistribution dist = lognormal_batch_pdf(1.0, 1.0, 32);
        const double sla_ms = derive_sla_target(table, 32, 1.5);
        for (int gpus : {1, 2}) {
            const ParisResult pr = paris_plan(table, dist, 7 * gpus, gpus, 7);
            // capacity-free rates: a light, a busy and an overloaded stream
            for (double rate : {200.0, 1500.0, 6000.0}) {
                const QueryTrace trace = sample_trace(dist, rate, 2000.0, 17 + case_id);
                for (SchedulerKind sk : {SchedulerKind::Elsa, SchedulerKind::Fifs}) {
                    EngineOptions opt;
                    opt.warmup_fraction = (case_id % 3) * 0.1;
                    opt.check_wait_consistency = (case_id % 2) == 0;
                    if (case_id % 4 == 1) {
                        opt.segment_routing = true;
                        opt.routing_segments = pr.segments;
                    }
                    const SimReport r = run(pr.plan, sk, trace, table, SlaConfig{sla_ms, 1.0, 1.0}, opt);
                    std::cout << "# case " << case_id << "\n";
                    write_query_csv(r, std::cout);
                    std::cout << report_to_json(r).dump() << "\n";
                    ++case_id;
                }
            }
        }
    }
    return 0;
}
