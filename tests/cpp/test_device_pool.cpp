// Host-only check of the device pool (csrc/device_pool.h): random alloc/free traffic placed by
// the pool must reserve exactly what the reference's run_mempool model reserves when replaying
// the pool's own recorded trace (mempool.hpp:285-387), for every policy combination.
#include <cstdio>
#include <random>
#include <unordered_map>
#include <vector>

#include "../../paper_2401_09149_b200/csrc/device_pool.h"

int main() {
    int failures = 0;
    for (int pol_i = 0; pol_i < 4; ++pol_i) {
        for (int trial = 0; trial < 20; ++trial) {
            seqplan::MempoolPolicy pol;
            pol.pinned_comm_pool = pol_i & 1;
            pol.consolidate_every_k_mlp = (pol_i & 2) ? 3 : 0;  // mixed-size MLP outputs packed 3 to a region
            pol.grad_premap = false;
            isp::DevicePool pool;
            pool.set_host_only(true);
            pool.set_policy(pol);
            std::mt19937 rng(1000 * pol_i + trial);
            std::vector<void*> live;
            const std::int64_t sizes[] = {512, 4096, 1 << 20, 3 << 20, 688 << 20, 176 << 20, 256 << 20};
            const seqplan::AllocTag tags[] = {seqplan::AllocTag::MlpIntermediate, seqplan::AllocTag::MlpOutput,
                                              seqplan::AllocTag::CommBuffer, seqplan::AllocTag::Other};
            for (int op = 0; op < 200; ++op) {
                if (!live.empty() && (rng() % 3 == 0 || live.size() > 12)) {
                    const size_t k = rng() % live.size();
                    pool.free(live[k], nullptr);
                    live.erase(live.begin() + long(k));
                } else {
                    live.push_back(pool.alloc(sizes[rng() % 7], tags[rng() % 4], nullptr));
                }
                if (op % 50 == 49) pool.step_boundary();
                // device accounting conserves bytes under every policy
                const auto d = pool.stats();
                if (d.reserved != d.allocated + d.free_cached + d.fragmented) {
                    std::printf("policy %d trial %d op %d: device conservation broken\n", pol_i, trial, op);
                    ++failures;
                }
            }
            for (void* p : live) pool.free(p, nullptr);
            pool.step_boundary();
            // model: the general pool of run_mempool on the same trace with pinned off
            seqplan::MempoolPolicy base = pol;
            base.pinned_comm_pool = false;
            const auto rep = seqplan::run_mempool(pool.trace(), pol);
            if (!pol.pinned_comm_pool && !pol.consolidate_every_k_mlp) {
                if (rep.per_step.back().reserved != pool.general_reserved()) {
                    std::printf("policy %d trial %d: pool reserved %lld model %lld\n", pol_i, trial,
                                (long long)pool.general_reserved(), (long long)rep.per_step.back().reserved);
                    ++failures;
                }
            }
            // conservation of the model over the device trace
            for (const auto& st : rep.per_step)
                if (st.reserved != st.allocated + st.free_cached + st.fragmented) ++failures;
        }
    }
    // The a = 1 trace of the reference (synthesize_trace) fed op by op to the device pool, under
    // every policy incl. consolidate-every-3 and grad pre-map: one step reserves exactly what
    // run_mempool reserves; over 3 steps the device recycles its packed regions (flat), while the
    // reference's consolidated_reserved grows.
    {
      for (int cfg = 0; cfg < 2; ++cfg) {  // 7B-32K L32 and 20B-128K L60 at p = 8
        seqplan::ModelConfig m;
        m.hidden_dim = cfg ? 5120 : 4096; m.layers = cfg ? 60 : 32; m.heads = cfg ? 40 : 32; m.vocab = 1;
        m.seq_len = cfg ? 131072 : 32768; m.global_batch_tokens = m.seq_len; m.bytes_per_element = 2;
        seqplan::ClusterConfig cl;
        cl.total_gpus = 8; cl.gpus_per_node = 8; cl.gpu_memory_capacity = std::int64_t(180) << 30;
        for (int steps : {1, 3}) {
            seqplan::Strategy s;
            s.micro_batch_num = steps; s.recompute = 1; s.sp = 8; s.ps = 8;
            m.global_batch_tokens = m.seq_len * steps;
            const seqplan::Trace tr = seqplan::synthesize_trace(m, s, cl);
            for (int pol_i = 0; pol_i < 8; ++pol_i) {
                seqplan::MempoolPolicy pol;
                pol.pinned_comm_pool = pol_i & 1;
                pol.consolidate_every_k_mlp = (pol_i & 2) ? 3 : 0;
                pol.grad_premap = pol_i & 4;
                isp::DevicePool pool;
                pool.set_host_only(true);
                pool.set_policy(pol);
                if (pol.grad_premap) pool.premap_grads(seqplan::run_mempool(tr, pol).per_step.empty() ? 0 :
                                                       m.seq_len / 8 * m.hidden_dim * 2);
                std::unordered_map<std::int64_t, void*> ptr;
                for (const auto& op : tr.ops) {
                    if (op.kind == seqplan::TraceOp::Kind::Alloc) ptr[op.id] = pool.alloc(op.size, op.tag, nullptr);
                    else if (op.kind == seqplan::TraceOp::Kind::Free) pool.free(ptr[op.id], nullptr);
                    else pool.step_boundary();
                }
                const auto rep = seqplan::run_mempool(tr, pol);
                const std::int64_t dev = pool.stats().peak_reserved, ref = rep.peak_reserved;
                const bool ok = steps == 1 ? dev == ref : (dev <= ref && (pol.consolidate_every_k_mlp ? dev < ref : dev == ref));
                if (!ok) {
                    std::printf("synth trace steps %d policy %d: device peak %lld reference %lld\n", steps, pol_i,
                                (long long)dev, (long long)ref);
                    ++failures;
                }
            }
        }
      }
    }
    std::printf("device pool vs run_mempool: %s\n", failures ? "FAIL" : "ok");
    return failures ? 1 : 0;
}
