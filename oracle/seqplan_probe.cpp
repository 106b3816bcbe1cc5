// seqplan_probe.cpp — dumps the layout / schedule / pool outputs of the seqplan
// API as JSON, for bit-exact parity between the reference headers and ours.
//
// ORACLE / TEST INFRASTRUCTURE ONLY. Compiled twice by oracle/Makefile:
//   -I /root/reference/proj/include  -> oracle/_ref/seqplan_probe  (the reference itself)
//   -I include                       -> built by tests/test_seqplan_golden.py
// The reference run is frozen into tests/golden/seqplan_golden.json (the GPU box
// has no /root/reference). Every probed function and its reference line:
//   ShardingLayout::make         strategy.hpp:52-62
//   validate                     strategy.hpp:72-99
//   place_groups                 placement.hpp:39-59
//   estimate_comm_layer          cost.hpp:160-206   (sp / ps branches on the ISP plan)
//   estimate_comp_layer          cost.hpp:224-241
//   estimate_memory              cost.hpp:124-150   (other_buffers = pinned double buffer)
//   estimate_step                cost.hpp:268-297   (OPro)
//   simulate_forward / backward  overlap_sim.hpp:80-153
//   compare_to_analytic          overlap_sim.hpp:165-173
//   synthesize_trace, run_mempool mempool.hpp:91-135, 285-387
#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <algorithm>
#include <vector>

#include "seqplan/cost.hpp"
#include "seqplan/mempool.hpp"
#include "seqplan/overlap_sim.hpp"
#include "seqplan/placement.hpp"
#include "seqplan/strategy.hpp"

using namespace seqplan;

namespace {

struct Out {
    bool first = true;
    void key(const char* k) {
        std::printf("%s\"%s\":", first ? "" : ",", k);
        first = false;
    }
};

void num(double v) { std::printf("%.17g", v); }
void inum(long long v) { std::printf("%lld", v); }

struct BlockCfg {
    const char* name;
    long long H, D, S, e;
};

const BlockCfg kConfigs[] = {
    {"cpu_ref_h512_s1k", 512, 8, 1024, 4},
    {"7b_s4k", 4096, 32, 4096, 2},
    {"7b_s32k", 4096, 32, 32768, 2},
    {"7b_s2k", 4096, 32, 2048, 2},
    {"20b_s128k", 5120, 40, 131072, 2},
};

ModelConfig block_model(const BlockCfg& c, long long layers = 1) {
    ModelConfig m;
    m.hidden_dim = c.H;
    m.layers = layers;
    m.heads = c.D;
    m.vocab = 1;
    m.seq_len = c.S;
    m.global_batch_tokens = c.S;
    m.bytes_per_element = c.e;
    return m;
}

Strategy isp(long long p, long long a = 0) {
    Strategy s;
    s.recompute = a;
    s.sp = p;
    s.ps = p;
    return s;
}

void dump_timeline(const Timeline& tl) {
    std::printf("{\"makespan\":");
    num(tl.makespan);
    std::printf(",\"events\":[");
    for (size_t i = 0; i < tl.events.size(); ++i) {
        const auto& e = tl.events[i];
        std::printf("%s[%d,\"%s\",%lld,", i ? "," : "", e.stream == StreamKind::Compute ? 0 : 1,
                    e.kind.c_str(), (long long)e.layer);
        num(e.start);
        std::printf(",");
        num(e.end);
        std::printf("]");
    }
    std::printf("]}");
}

void dump_report(const FragmentationReport& r) {
    std::printf("{\"peak_reserved\":%lld,\"peak_fragmented\":%lld,\"final_fragmented\":%lld,"
                "\"fragment_threshold\":%lld,\"oom_events\":%lld,\"per_step\":[",
                (long long)r.peak_reserved, (long long)r.peak_fragmented, (long long)r.final_fragmented,
                (long long)r.fragment_threshold, (long long)r.oom_events);
    for (size_t i = 0; i < r.per_step.size(); ++i) {
        const auto& s = r.per_step[i];
        std::printf("%s[%lld,%lld,%lld,%lld]", i ? "," : "", (long long)s.reserved, (long long)s.allocated,
                    (long long)s.free_cached, (long long)s.fragmented);
    }
    std::printf("],\"peak_fragment_sizes\":{");
    bool f = true;
    for (const auto& [size, count] : r.peak_fragment_sizes) {
        std::printf("%s\"%lld\":%lld", f ? "" : ",", (long long)size, (long long)count);
        f = false;
    }
    std::printf("}}");
}

// --time <config>: the reference's own CPU path for one block of the config, timed on this host
// (bench.py's cpu_baseline): estimate_step at p = 1, 2, 4, 8 (cost.hpp:268-297),
// simulate_forward(InterLayerPrefetch) + simulate_backward(Selective) of a 32-layer workload built
// from the block's own prices (overlap_sim.hpp:80-153), synthesize_trace + run_mempool (all
// policies on) of the 32-layer a = 1 trace at p = 8 (mempool.hpp:91-135, 285-387). Microseconds
// per call, median of 7 repetitions of a loop sized to ~20 ms.
template <class F>
double time_us(F&& f) {
    using clk = std::chrono::steady_clock;
    int iters = 1;
    for (;;) {
        auto t0 = clk::now();
        for (int i = 0; i < iters; ++i) f();
        const double dt = std::chrono::duration<double>(clk::now() - t0).count();
        if (dt > 0.02 || iters > (1 << 24)) break;
        iters *= 2;
    }
    std::vector<double> v;
    for (int r = 0; r < 7; ++r) {
        auto t0 = clk::now();
        for (int i = 0; i < iters; ++i) f();
        v.push_back(std::chrono::duration<double>(clk::now() - t0).count() * 1e6 / iters);
    }
    std::sort(v.begin(), v.end());
    return v[3];
}

volatile double g_sink = 0;

int time_config(const char* name) {
    const BlockCfg* c = nullptr;
    for (const auto& k : kConfigs)
        if (!std::strcmp(k.name, name)) c = &k;
    if (!c) return 2;
    const BandwidthProfile flat = BandwidthProfile::flat(900e9);
    ComputeModel cm;
    cm.peak_flops_per_gpu = 1656.3e12;
    cm.efficiency = 1.0;
    OverlapModel om;
    std::printf("{\"config\":\"%s\"", c->name);
    for (long long p : {1LL, 2LL, 4LL, 8LL}) {
        const ModelConfig m = block_model(*c);
        ClusterConfig cl{p, p < 8 ? p : 8, 192LL << 30};
        const Strategy s = isp(p);
        std::printf(",\"estimate_step_p%lld_us\":", p);
        num(time_us([&] { g_sink = g_sink + estimate_step(s, m, cl, flat, cm, om).t_step; }));
    }
    {  // 32 layers with this block's p = 8 prices (fwd compute, gather, bwd G-X / G-W, RS)
        const ModelConfig m = block_model(*c);
        ClusterConfig cl{8, 8, 192LL << 30};
        const Strategy s = isp(8);
        auto pl = place_groups(cl, s);
        const auto comm = estimate_comm_layer(s, m, cl, pl, flat);
        const double comp = estimate_comp_layer(s, m, cm);
        const double ag = comm.ps / 3.0;
        std::vector<LayerWorkload> layers(32, LayerWorkload{comp / 3.0, ag, comp / 3.0, comp / 3.0, ag});
        std::printf(",\"simulate_fwd_bwd_L32_us\":");
        num(time_us([&] {
            g_sink = g_sink + simulate_forward(layers, ForwardPolicy::InterLayerPrefetch, 0.0).makespan +
                     simulate_backward(layers, BackwardPolicy::Selective, 0.0).makespan;
        }));
    }
    {
        ModelConfig m = block_model(*c, 32);
        Strategy s = isp(8, 1);
        ClusterConfig cl{8, 8, 192LL << 30};
        auto trace = synthesize_trace(m, s, cl);
        MempoolPolicy pol;
        pol.pinned_comm_pool = true;
        pol.consolidate_every_k_mlp = 3;
        pol.grad_premap = true;
        pol.capacity = 192LL << 30;
        std::printf(",\"run_mempool_L32_p8_us\":");
        num(time_us([&] { g_sink = g_sink + (double)run_mempool(trace, pol).peak_reserved; }));
        std::printf(",\"trace_ops\":%zu", trace.ops.size());
    }
    std::printf(",\"threads\":1}\n");
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc == 3 && !std::strcmp(argv[1], "--time")) return time_config(argv[2]);
    Out o;
    std::printf("{");

    // ---- layouts: per-tensor shards of the SwiGLU block and the Psi_ref shard ----
    o.key("layouts");
    std::printf("{");
    bool f1 = true;
    for (const auto& c : kConfigs) {
        const long long I = mlp_intermediate_dim(c.H);
        const long long numel[7] = {c.H, 3 * c.H * c.H, c.H * c.H, c.H, I * c.H, I * c.H, c.H * I};
        for (long long p : {1LL, 2LL, 4LL, 8LL}) {
            std::printf("%s\"%s/p%lld\":[", f1 ? "" : ",", c.name, p);
            f1 = false;
            for (int t = 0; t < 7; ++t) {
                auto l = ShardingLayout::make(numel[t], p, p);
                std::printf("%s[%lld,%lld,%lld]", t ? "," : "", (long long)l.factor,
                            (long long)l.replica_groups, (long long)l.elements_per_gpu);
            }
            auto lr = ShardingLayout::make(layer_param_count(block_model(c)), p, p);
            std::printf(",[%lld,%lld,%lld],%lld]", (long long)lr.factor, (long long)lr.replica_groups,
                        (long long)lr.elements_per_gpu, (long long)I);
        }
    }
    std::printf("}");

    // ---- validate + place_groups + prices at every config and p ----
    o.key("plans");
    std::printf("{");
    bool f2 = true;
    const BandwidthProfile flat = BandwidthProfile::flat(900e9);
    ComputeModel cm;
    cm.peak_flops_per_gpu = 1656.3e12;
    cm.efficiency = 1.0;
    OverlapModel om;
    for (const auto& c : kConfigs) {
        for (long long p : {1LL, 2LL, 4LL, 8LL}) {
            const ModelConfig m = block_model(c);
            ClusterConfig cl{p, p < 8 ? p : 8, 192LL << 30};
            const Strategy s = isp(p);
            std::printf("%s\"%s/p%lld\":{", f2 ? "" : ",", c.name, p);
            f2 = false;
            auto v = validate(s, m, cl);
            std::printf("\"valid\":%s,", v.ok() ? "true" : "false");
            auto pl = place_groups(cl, s);
            std::printf("\"axes\":[%d,%d,%d,%d,%d],", (int)pl[GroupKind::TpSp], (int)pl[GroupKind::Ps],
                        (int)pl[GroupKind::Oss], (int)pl[GroupKind::Gs], (int)pl[GroupKind::Dp]);
            auto comm = estimate_comm_layer(s, m, cl, pl, flat);
            std::printf("\"comm\":[");
            num(comm.tp); std::printf(","); num(comm.sp); std::printf(","); num(comm.ps);
            std::printf(","); num(comm.oss); std::printf(","); num(comm.gs);
            std::printf("],\"comp\":");
            num(estimate_comp_layer(s, m, cm));
            auto mem = estimate_memory(s, m, cl);
            std::printf(",\"other_buffers\":");
            num(mem.other_buffers);
            std::printf(",\"act\":");
            num(mem.act);
            auto st = estimate_step(s, m, cl, flat, cm, om);
            std::printf(",\"opro\":");
            num(st.t_layer_overlapped);
            std::printf(",\"t_step\":");
            num(st.t_step);
            std::printf("}");
        }
    }
    // a few infeasible ISP plans (head divisibility / GPU count)
    {
        ModelConfig m = block_model(kConfigs[1]);
        m.heads = 12;
        ClusterConfig cl{8, 8, 0};
        auto v = validate(isp(8), m, cl);
        std::printf(",\"infeasible_heads12_p8\":{\"valid\":%s,\"n\":%zu}", v.ok() ? "true" : "false",
                    v.violations.size());
    }
    std::printf("}");

    // ---- overlap schedules ----
    o.key("schedules");
    std::printf("{");
    {
        std::mt19937 rng(2401);
        std::uniform_real_distribution<double> d(0.1, 20.0);
        for (int trial = 0; trial < 24; ++trial) {
            std::vector<LayerWorkload> layers(1 + trial % 6);
            for (auto& w : layers) w = LayerWorkload{d(rng), d(rng), d(rng), d(rng), d(rng)};
            const double delay = (trial % 3 == 0) ? 0.25 : 0.0;
            std::printf("%s\"t%d\":{\"fwd_naive\":", trial ? "," : "", trial);
            dump_timeline(simulate_forward(layers, ForwardPolicy::Naive, delay));
            std::printf(",\"fwd_prefetch\":");
            dump_timeline(simulate_forward(layers, ForwardPolicy::InterLayerPrefetch, delay));
            std::printf(",\"bwd_fused\":");
            dump_timeline(simulate_backward(layers, BackwardPolicy::Fused, delay));
            auto sel = simulate_backward(layers, BackwardPolicy::Selective, delay);
            std::printf(",\"bwd_selective\":");
            dump_timeline(sel);
            auto r = compare_to_analytic(sel, 1.3);
            std::printf(",\"analytic\":[");
            num(r.makespan); std::printf(","); num(r.total_compute); std::printf(",");
            num(r.total_comm); std::printf(","); num(r.analytic); std::printf(","); num(r.ratio);
            std::printf("]}");
        }
    }
    std::printf("}");

    // ---- pool traces (a = 1, ISP plan at p = 8; 65B-style long sequence) ----
    o.key("pools");
    std::printf("{");
    {
        struct PoolCase { const char* name; long long H, D, S, L, p, n; };
        const PoolCase cases[] = {
            {"7b_s32k_L32_p8", 4096, 32, 32768, 32, 8, 1},
            {"20b_s128k_L60_p8", 5120, 40, 131072, 60, 8, 1},
            {"7b_s4k_L8_p4_n2", 4096, 32, 4096, 8, 4, 2},
            {"65b_s16k_L8_p1", 8192, 64, 16384, 8, 1, 1},
            {"cpu_ref_L4_p2", 512, 8, 1024, 4, 2, 1},
        };
        MempoolPolicy pols[5];
        pols[1].pinned_comm_pool = true;
        pols[2].consolidate_every_k_mlp = 3;
        pols[3].grad_premap = true;
        pols[4].pinned_comm_pool = true;
        pols[4].consolidate_every_k_mlp = 3;
        pols[4].grad_premap = true;
        const char* pol_names[5] = {"base", "pinned", "consolidate3", "premap", "all"};
        bool f3 = true;
        for (const auto& pc : cases) {
            ModelConfig m;
            m.hidden_dim = pc.H;
            m.layers = pc.L;
            m.heads = pc.D;
            m.vocab = 1;
            m.seq_len = pc.S;
            m.global_batch_tokens = pc.S * pc.n;
            Strategy s = isp(pc.p, 1);
            s.micro_batch_num = pc.n;
            ClusterConfig cl{pc.p, pc.p, 192LL << 30};
            auto trace = synthesize_trace(m, s, cl);
            std::printf("%s\"%s\":{\"ops\":%zu", f3 ? "" : ",", pc.name, trace.ops.size());
            f3 = false;
            for (int k = 0; k < 5; ++k) {
                std::printf(",\"%s\":", pol_names[k]);
                MempoolPolicy pol = pols[k];
                pol.capacity = 4LL << 30;
                dump_report(run_mempool(trace, pol));
            }
            std::printf("}");
        }
    }
    std::printf("}");
    std::printf("}\n");
    return 0;
}
