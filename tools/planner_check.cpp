// planner_check.cpp — closes the loop from measured B200 profiles back into the planner
// (SURVEY.md §8(f) item 1).
//
// Reads a VPro bandwidth CSV in the reference's format (bandwidth.hpp:214-253) and a measured
// UPro per-layer forward time, prices the ISP plan with the reference's estimate_step
// (cost.hpp:268-297) and prints predicted vs measured per-layer fwd+bwd time, plus the overlap
// slowdown ratio R that would make the analytic OPro match the measurement.
//   planner_check <vpro.csv> <H> <heads> <S> <p> <fwd_compute_s> <measured_step_s>
#include <cstdio>
#include <cstdlib>
#include <fstream>

#include "seqplan/cost.hpp"

int main(int argc, char** argv) {
    if (argc < 8) {
        std::fprintf(stderr, "usage: %s vpro.csv H heads S p fwd_compute_s measured_step_s\n", argv[0]);
        return 2;
    }
    using namespace seqplan;
    const BandwidthProfile prof = load_bandwidth_csv_file(argv[1]);
    ModelConfig m;
    m.hidden_dim = std::atoll(argv[2]);
    m.heads = std::atoll(argv[3]);
    m.seq_len = std::atoll(argv[4]);
    m.layers = 1;
    m.vocab = 1;
    m.global_batch_tokens = m.seq_len;
    const std::int64_t p = std::atoll(argv[5]);
    const double fwd_s = std::atof(argv[6]);
    const double measured = std::atof(argv[7]);
    Strategy s;
    s.sp = p;
    s.ps = p;
    ClusterConfig cl{p, p, 192LL << 30};
    ComputeModel cm;
    cm.mode = ComputeModel::Mode::Profiled;  // UPro: measured forward time of this block
    cm.layer_forward_s[{1, m.seq_len / p, 1}] = fwd_s;
    const CostBreakdown c = estimate_step(s, m, cl, prof, cm, OverlapModel{});
    const double comm = c.comm.recurring();
    const double comp = c.t_comp_per_layer;
    const double r_fit = measured / std::max(comm, comp);
    std::printf("{\"p\": %lld, \"comm_sp_s\": %.6g, \"comm_ps_s\": %.6g, \"comp_s\": %.6g, \"opro_R1.30_s\": %.6g, "
                "\"measured_s\": %.6g, \"pred_over_measured\": %.4f, \"R_fit\": %.4f}\n",
                (long long)p, c.comm.sp, c.comm.ps, comp, c.t_layer_overlapped, measured,
                c.t_layer_overlapped / measured, r_fit);
    return 0;
}
