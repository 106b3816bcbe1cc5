// isp_block_demo.cpp — a seqplan-side caller of the B200 executor (single GPU, p = 1).
//
// Drives one ISP block fwd+bwd through seqplan::IspBlock (include/seqplan/isp_block.hpp), then
// feeds the measured CUDA-event schedule back into the reference's own analysis function
// compare_to_analytic (overlap_sim.hpp:165-173) and prints the device pool's StepStats.
// Build: see tests/test_cpp_frontend.py (g++ -std=c++20 ... -lseqplan_isp -lcudart).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "seqplan/isp_block.hpp"

int main(int argc, char** argv) {
    seqplan::ModelConfig m;
    m.hidden_dim = argc > 1 ? std::atoll(argv[1]) : 1024;
    m.heads = argc > 2 ? std::atoll(argv[2]) : 8;
    m.seq_len = argc > 3 ? std::atoll(argv[3]) : 2048;
    m.layers = 1;
    m.vocab = 1;
    m.global_batch_tokens = m.seq_len;
    const seqplan::Strategy s = seqplan::Strategy::isp(1);
    seqplan::IspBlock blk(m, s, /*rank=*/0, /*device=*/0, seqplan::IspBlock::default_policy(), SEQPLAN_ISP_FLAG_TIMELINE);
    blk.init_weights(0x5EED2401ull);
    const size_t bytes = size_t(m.seq_len) * size_t(m.hidden_dim) * 2;
    void *x = nullptr, *y = nullptr, *dx = nullptr;
    cudaMalloc(&x, bytes);
    cudaMalloc(&y, bytes);
    cudaMalloc(&dx, bytes);
    seqplan_isp_fill_activation(blk.handle(), 0x5EED2401ull, 0, x, nullptr);
    for (int it = 0; it < 3; ++it) {
        blk.forward(x, y);
        blk.backward(x, dx);  // dy := x (any bf16 tensor of the right shape)
    }
    cudaDeviceSynchronize();
    const seqplan::Timeline tl = blk.timeline();
    const seqplan::OverlapRatioReport r = seqplan::compare_to_analytic(tl, 1.30);
    const seqplan::StepStats st = blk.pool_stats();
    std::printf("{\"events\": %zu, \"makespan_ms\": %.4f, \"compute_ms\": %.4f, \"comm_ms\": %.4f, "
                "\"analytic_ms\": %.4f, \"ratio\": %.4f, \"exposed_comm_ms\": %.4f, "
                "\"pool_reserved\": %lld, \"pool_allocated\": %lld, \"pool_fragmented\": %lld}\n",
                tl.events.size(), r.makespan * 1e3, r.total_compute * 1e3, r.total_comm * 1e3, r.analytic * 1e3,
                r.ratio, seqplan::exposed_comm(tl) * 1e3, (long long)st.reserved, (long long)st.allocated,
                (long long)st.fragmented);
    try {
        seqplan::Strategy bad = s;
        bad.tp = 2;  // not the ISP plan: must surface as std::invalid_argument
        seqplan::IspBlock nope(m, bad, 0, 0);
        std::printf("ERROR: invalid plan accepted\n");
        return 1;
    } catch (const std::invalid_argument&) {
    }
    cudaFree(x);
    cudaFree(y);
    cudaFree(dx);
    return 0;
}
