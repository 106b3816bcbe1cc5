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

    /// The reference's model of this pool: run_mempool over the device pool's own recorded trace
    /// (mempool.hpp:285-387); peak_reserved / peak_fragmented cover the whole trace.
    FragmentationReport pool_replay() const {
        seqplan_step_stats s{};
        std::int64_t n = 0;
        raise(seqplan_isp_pool_replay(ctx_, &s, &n));
        FragmentationReport r;
        r.peak_reserved = s.peak_reserved;
        r.peak_fragmented = s.peak_fragmented;
        StepStats last;
        last.reserved = s.reserved;
        last.allocated = s.allocated;
        last.free_cached = s.free_cached;
        last.fragmented = s.fragmented;
        r.per_step.push_back(last);
        r.final_fragmented = s.fragmented;
        return r;
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
        if (status == SEQPLAN_ISP_ERR_INVALID || status == SEQPLAN_ISP_ERR_UNSUPPORTED) throw std::invalid_argument(msg);
        throw std::runtime_error(msg + " (status " + std::to_string(status) + ")");
    }

    seqplan_isp_ctx* ctx_ = nullptr;
};

/// ModelConfig::layers ISP blocks run as one step (seqplan_isp_stack_*): every forward gather
/// issued up front and the backward re-gathers in reverse layer order on one comm stream
/// (overlap_sim.hpp:80-153), one device pool for all layers (checkpoints between layers are
/// MlpOutput allocations, mempool.hpp:91-135); Strategy::recompute = 1 re-runs each layer's
/// forward in its backward.
class IspStack {
public:
    IspStack(const ModelConfig& model, const Strategy& s, int rank, int device,
             const MempoolPolicy& policy = IspBlock::default_policy(), std::uint32_t flags = 0) {
        if (model.layers < 1) throw std::invalid_argument("IspStack needs at least one layer");
        seqplan_isp_shape sh{model.hidden_dim, model.heads, model.seq_len, 0, 10000.0, 1e-5};
        seqplan_strategy st{s.micro_batch, s.micro_batch_num, s.recompute, s.pp, s.dp,
                            s.tp, s.sp, s.ps, s.gs, s.oss};
        seqplan_mempool_policy p{policy.pinned_comm_pool ? 1 : 0, policy.consolidate_every_k_mlp,
                                 policy.grad_premap ? 1 : 0, policy.capacity};
        const int status = seqplan_isp_stack_create(static_cast<int>(model.layers), static_cast<int>(s.sp), rank,
                                                    device, &sh, &st, &p, flags, &stack_);
        if (status == SEQPLAN_ISP_ERR_INVALID) throw std::invalid_argument("seqplan_isp_stack_create: invalid plan");
        if (status != SEQPLAN_ISP_OK)
            throw std::runtime_error("seqplan_isp_stack_create failed (status " + std::to_string(status) + ")");
    }
    IspStack(const IspStack&) = delete;
    IspStack& operator=(const IspStack&) = delete;
    ~IspStack() { seqplan_isp_stack_destroy(stack_); }

    int layers() const { return seqplan_isp_stack_layers(stack_); }
    /// Layer l's context (weights, gradient shards, peer bootstrap); owned by the stack.
    seqplan_isp_ctx* layer(int l) const { return seqplan_isp_stack_layer(stack_, l); }

    void forward(const void* x, void* y, void* stream = nullptr) { check(seqplan_isp_stack_fwd(stack_, x, y, stream)); }
    void backward(const void* dy, void* dx, void* stream = nullptr) {
        check(seqplan_isp_stack_bwd(stack_, dy, dx, stream));
    }

private:
    void check(int status) const {
        if (status == SEQPLAN_ISP_OK) return;
        seqplan_isp_ctx* c = seqplan_isp_stack_layer(stack_, 0);
        const std::string msg = c ? seqplan_isp_last_error(c) : "seqplan_isp_stack";
        if (status == SEQPLAN_ISP_ERR_INVALID || status == SEQPLAN_ISP_ERR_UNSUPPORTED) throw std::invalid_argument(msg);
        throw std::runtime_error(msg + " (status " + std::to_string(status) + ")");
    }

    seqplan_isp_stack* stack_ = nullptr;
};

}  // namespace seqplan
