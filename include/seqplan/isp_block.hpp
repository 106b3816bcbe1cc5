// seqplan/isp_block.hpp — C++ front-end of the B200 ISP block executor.
//
// Wraps the C ABI of include/seqplan_isp.h in the reference's own vocabulary so a
// seqplan-based caller drives the executor with ModelConfig / Strategy / MempoolPolicy
// (model.hpp:12-48, strategy.hpp:16-48, mempool.hpp:137-142) and gets its measured
// behaviour back as the reference's types: the CUDA-event schedule as a Timeline
// (overlap_sim.hpp:28-46, so compare_to_analytic at overlap_sim.hpp:165-173 applies
// unchanged) and pool statistics as StepStats. Status codes map back to the
// reference's exception classes: invalid argument -> std::invalid_argument,
// everything else -> std::runtime_error.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "seqplan/mempool.hpp"
#include "seqplan/model.hpp"
#include "seqplan/overlap_sim.hpp"
#include "seqplan/strategy.hpp"
#include "seqplan_isp.h"

namespace seqplan {

class IspBlock {
public:
    /// One rank of the ISP plan s (sp = ps = world); throws std::invalid_argument for a plan
    /// the reference's validate() rejects or that is not the ISP plan.
    IspBlock(const ModelConfig& model, const Strategy& s, int rank, int device,
             const MempoolPolicy& policy = default_policy(), std::uint32_t flags = 0) {
        seqplan_isp_shape sh{model.hidden_dim, model.heads, model.seq_len, 0, 10000.0, 1e-5};
        seqplan_strategy st{s.micro_batch, s.micro_batch_num, s.recompute, s.pp, s.dp,
                            s.tp, s.sp, s.ps, s.gs, s.oss};
        seqplan_mempool_policy p{policy.pinned_comm_pool ? 1 : 0, policy.consolidate_every_k_mlp,
                                 policy.grad_premap ? 1 : 0, policy.capacity};
        raise(seqplan_isp_ctx_create(static_cast<int>(s.sp), rank, device, &sh, &st, &p, flags, &ctx_));
    }
    IspBlock(const IspBlock&) = delete;
    IspBlock& operator=(const IspBlock&) = delete;
    ~IspBlock() { seqplan_isp_ctx_destroy(ctx_); }

    static MempoolPolicy default_policy() {
        MempoolPolicy p;
        p.pinned_comm_pool = true;
        p.grad_premap = true;
        return p;
    }

    seqplan_isp_ctx* handle() const { return ctx_; }

    void init_weights(std::uint64_t seed) { raise(seqplan_isp_init_weights(ctx_, seed)); }
    void forward(const void* x, void* y, void* stream = nullptr) { raise(seqplan_isp_block_fwd(ctx_, x, y, stream)); }
    void backward(const void* dy, void* dx, void* stream = nullptr) {
        raise(seqplan_isp_block_bwd(ctx_, dy, dx, stream));
    }
    std::vector<float> grad_shard(int tensor) {
        std::vector<float> out(static_cast<std::size_t>(seqplan_isp_shard_numel(ctx_, tensor)));
        raise(seqplan_isp_get_grad_shard(ctx_, tensor, out.data(), static_cast<std::int64_t>(out.size())));
        return out;
    }

    /// Pool statistics of the device pool as the reference's StepStats.
    StepStats pool_stats() const {
        seqplan_step_stats s{};
        raise(seqplan_isp_pool_stats(ctx_, &s));
        StepStats out;
        out.reserved = s.reserved;
        out.allocated = s.allocated;
        out.free_cached = s.free_cached;
        out.fragmented = s.fragmented;
        return out;
    }

    /// The last fwd+bwd as a reference Timeline (needs SEQPLAN_ISP_FLAG_TIMELINE). Module
    /// index plays the role of the layer; all-to-all events run on the compute stream.
    Timeline timeline() const {
        std::int64_t n = 0;
        raise(seqplan_isp_timeline(ctx_, nullptr, &n));
        std::vector<seqplan_timeline_event> ev(static_cast<std::size_t>(n));
        raise(seqplan_isp_timeline(ctx_, ev.data(), &n));
        static const char* const kinds[] = {"forward", "grad_input", "grad_weight", "all_gather",
                                            "reduce_scatter", "all_to_all"};
        Timeline tl;
        for (const auto& e : ev) {
            tl.events.push_back(TimelineEvent{e.stream == 0 ? StreamKind::Compute : StreamKind::Comm,
                                              kinds[e.kind], e.layer, e.start_s, e.end_s});
            tl.makespan = std::max(tl.makespan, e.end_s);
        }
        return tl;
    }

private:
    void raise(int status) const {
        if (status == SEQPLAN_ISP_OK) return;
        const std::string msg = ctx_ ? seqplan_isp_last_error(ctx_) : "seqplan_isp_ctx_create failed";
        if (status == SEQPLAN_ISP_ERR_INVALID) throw std::invalid_argument(msg);
        throw std::runtime_error(msg + " (status " + std::to_string(status) + ")");
    }

    seqplan_isp_ctx* ctx_ = nullptr;
};

}  // namespace seqplan
