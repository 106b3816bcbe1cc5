// Host-only check of the device pool (csrc/device_pool.h): random alloc/free traffic placed by
// the pool must reserve exactly what the reference's run_mempool model reserves when replaying
// the pool's own recorded trace (mempool.hpp:285-387), for every policy combination.
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2401_09149_b200/csrc/device_pool.h"

int main() {
    int failures = 0;
    for (int pol_i = 0; pol_i < 4; ++pol_i) {
        for (int trial = 0; trial < 20; ++trial) {
            seqplan::MempoolPolicy pol;
            pol.pinned_comm_pool = pol_i & 1;
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
            }
            for (void* p : live) pool.free(p, nullptr);
            pool.step_boundary();
            // model: the general pool of run_mempool on the same trace with pinned off
            seqplan::MempoolPolicy base = pol;
            base.pinned_comm_pool = false;
            const auto rep = seqplan::run_mempool(pool.trace(), pol);
            if (!pol.pinned_comm_pool) {
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
    std::printf("device pool vs run_mempool: %s\n", failures ? "FAIL" : "ok");
    return failures ? 1 : 0;
}
