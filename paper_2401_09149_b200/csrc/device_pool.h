// Device memory pool of the ISP executor (north-star subsystem 5).
//
// Placement is the reference's best-fit caching pool, seqplan::detail::CachingPool
// (proj/include/seqplan/mempool.hpp:168-273): the smallest free chunk that fits,
// split at the chunk start, coalesce on free, segments reserved with exactly the
// request size and never released while the context lives. The policy knobs are
// MempoolPolicy's (mempool.hpp:137-142):
//   pinned_comm_pool : comm buffers (gathered weights) rotate through a dedicated
//                      double buffer (the first request reserves 2 slots of its size, more
//                      slots only when every slot is busy or too small), never touching the
//                      general pool (cost.hpp:147 other_buffers);
//   consolidate_every_k_mlp : MLP outputs (the per-layer checkpoints of the a = 1 regime) are
//                      packed k to a region of k x size (mempool.hpp:345-352). The reference
//                      never returns a packed region (its consolidated_reserved grows every
//                      step); here a region whose k slots are all free is
//                      recycled by the next packed request of the same size. Within one step
//                      the two agree byte for byte; across steps the device stays flat;
//   grad_premap      : gradient shards live in one arena reserved up front;
//   capacity         : reserved bytes above it count as OOM events.
// Every alloc/free is recorded as a seqplan::Trace, so run_mempool(trace, policy)
// replays the device pool bit-exactly (tests/test_device_pool.py).
//
// Stream safety: a freed chunk remembers the event recorded on the freeing stream;
// an allocation on another stream that reuses any byte of it waits on that event.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "seqplan/mempool.hpp"

namespace isp {

class DevicePool {
public:
    struct Stats {
        std::int64_t reserved = 0, allocated = 0, free_cached = 0, fragmented = 0;
        std::int64_t peak_reserved = 0, peak_fragmented = 0, peak_allocated = 0;
    };

    DevicePool() = default;
    DevicePool(const DevicePool&) = delete;
    DevicePool& operator=(const DevicePool&) = delete;
    ~DevicePool() { release_all(); }

    void set_policy(const seqplan::MempoolPolicy& p) { policy_ = p; }
    const seqplan::MempoolPolicy& policy() const { return policy_; }
    // Host-only mode (tests on CPU): no device memory is touched, addresses are offsets.
    void set_host_only(bool v) { host_only_ = v; }

    // Reserve the gradient arena up front (grad_premap).
    bool premap_grads(std::int64_t bytes) {
        if (!policy_.grad_premap || bytes <= 0) return true;
        if (!reserve_raw(bytes, &grad_arena_)) return false;
        grad_arena_bytes_ = bytes;
        return true;
    }

    void* alloc(std::int64_t bytes, seqplan::AllocTag tag, cudaStream_t stream) {
        bytes = round_up(bytes);
        const std::int64_t id = next_id_++;
        trace_.ops.push_back(seqplan::TraceOp::alloc(id, bytes, tag));
        if (++size_seen_[bytes] == 2 && (threshold_ == 0 || bytes < threshold_)) threshold_ = bytes;
        void* ptr = nullptr;
        Live lv{id, bytes, tag, Where::General, 0, 0};
        if (policy_.pinned_comm_pool && tag == seqplan::AllocTag::CommBuffer) {
            ptr = pinned_alloc(bytes, stream, lv);
        } else if (policy_.consolidate_every_k_mlp > 0 && tag == seqplan::AllocTag::MlpOutput) {
            ptr = packed_alloc(bytes, stream, lv);
            if (!ptr) return nullptr;
        } else if (policy_.grad_premap && tag == seqplan::AllocTag::Grad && grad_arena_) {
            if (grad_used_ + bytes > grad_arena_bytes_) return fail("grad arena exhausted");
            ptr = static_cast<char*>(grad_arena_) + grad_used_;
            lv.where = Where::Grad;
            lv.offset = grad_used_;
            grad_used_ += bytes;
            grad_alloc_ += bytes;
            ++grad_live_;
        } else {
            const bool fresh = pool_.alloc(id, bytes);
            const auto w = pool_.where(id);
            if (fresh) {
                void* seg = nullptr;
                if (!reserve_raw(bytes, &seg)) {
                    pool_.free(id);
                    return fail("device allocation failed");
                }
                segments_.push_back(seg);
            }
            ptr = static_cast<char*>(segments_[w.segment]) + w.offset;
            lv.where = Where::General;
            lv.segment = w.segment;
            lv.offset = w.offset;
            wait_for_reuse(lv, stream);
        }
        live_[ptr] = lv;
        snapshot();
        return ptr;
    }

    void free(void* ptr, cudaStream_t stream) {
        auto it = live_.find(ptr);
        if (it == live_.end()) return;
        const Live lv = it->second;
        live_.erase(it);
        trace_.ops.push_back(seqplan::TraceOp::free(lv.id));
        switch (lv.where) {
            case Where::General:
                pool_.free(lv.id);
                record_release(lv, stream);
                break;
            case Where::Pinned:
                pinned_alloc_ -= lv.bytes;
                record_pinned_release(lv, stream);
                break;
            case Where::Grad:
                grad_alloc_ -= lv.bytes;
                if (--grad_live_ == 0) grad_used_ = 0;  // bump arena: rewinds when empty
                break;
            case Where::Packed: {
                Region& r = regions_[lv.segment];
                r.used[static_cast<std::size_t>(lv.offset)] = false;
                packed_alloc_ -= lv.bytes;
                if (!host_only_) {
                    cudaEventRecord(r.ev, stream);
                    r.ev_valid = true;
                    r.last_stream = stream;
                }
                break;
            }
        }
        snapshot();
    }

    void step_boundary() {
        trace_.ops.push_back(seqplan::TraceOp::step_boundary());
        per_step_.push_back(snapshot());
    }

    // Device truth: bytes actually reserved / live right now, with peaks.
    Stats stats() const { return stats_; }
    // The reference model of this exact trace (mempool.hpp:285-387).
    seqplan::FragmentationReport replay() const { return seqplan::run_mempool(trace_, policy_); }
    std::int64_t general_reserved() const { return pool_.reserved(); }
    const seqplan::Trace& trace() const { return trace_; }
    const std::string& error() const { return error_; }
    std::int64_t segments() const { return static_cast<std::int64_t>(segments_.size()); }

    void release_all() {
        if (!host_only_) {
            for (void* s : segments_) cudaFree(s);
            for (auto& s : pinned_slots_) if (s.ptr) cudaFree(s.ptr);
            if (grad_arena_) cudaFree(grad_arena_);
            for (auto& e : pending_) cudaEventDestroy(e.ev);
            for (auto& s : pinned_slots_) if (s.ev) cudaEventDestroy(s.ev);
            for (auto& r : regions_) {
                if (r.ptr) cudaFree(r.ptr);
                if (r.ev) cudaEventDestroy(r.ev);
            }
        }
        regions_.clear();
        open_ = -1;
        segments_.clear();
        pinned_slots_.clear();
        pending_.clear();
        grad_arena_ = nullptr;
    }

private:
    enum class Where { General, Pinned, Grad, Packed };
    struct Live {
        std::int64_t id, bytes;
        seqplan::AllocTag tag;
        Where where;
        std::size_t segment;
        std::int64_t offset;
    };
    struct Pending {  // freed general-pool range still possibly in use on `stream`
        std::size_t segment;
        std::int64_t lo, hi;
        cudaStream_t stream;
        cudaEvent_t ev;
    };
    struct PinnedSlot {
        void* ptr = nullptr;
        std::int64_t bytes = 0;
        bool busy = false;
        cudaStream_t last_stream = nullptr;
        cudaEvent_t ev = nullptr;
        bool ev_valid = false;
    };

    struct Region {  // consolidated MLP-output region: k slots of `slot` bytes
        void* ptr = nullptr;
        std::int64_t slot = 0;
        std::vector<bool> used;
        std::int64_t handed_out = 0;  // slots ever handed out (the reference's packed_slots)
        cudaStream_t last_stream = nullptr;
        cudaEvent_t ev = nullptr;
        bool ev_valid = false;
    };

    static std::int64_t round_up(std::int64_t b) { return (b + 511) / 512 * 512; }

    void* fail(const char* why) {
        error_ = why;
        return nullptr;
    }

    bool reserve_raw(std::int64_t bytes, void** out) {
        if (host_only_) {
            *out = reinterpret_cast<void*>(static_cast<std::uintptr_t>(0x100000000ull + host_cursor_));
            host_cursor_ += round_up(bytes) + 4096;
            return true;
        }
        return cudaMalloc(out, static_cast<size_t>(bytes)) == cudaSuccess;
    }

    // Pinned comm double buffer: two slots sized by the largest request seen.
    void* pinned_alloc(std::int64_t bytes, cudaStream_t stream, Live& lv) {
        lv.where = Where::Pinned;
        PinnedSlot* slot = nullptr;
        for (auto& s : pinned_slots_)  // best fit among idle slots
            if (!s.busy && s.bytes >= bytes && (!slot || s.bytes < slot->bytes)) slot = &s;
        if (!slot) {
            // grow: a new slot only when every existing one is busy or too small
            pinned_slots_.push_back(PinnedSlot{});
            slot = &pinned_slots_.back();
            if (!reserve_raw(bytes, &slot->ptr)) return fail("pinned comm slot allocation failed");
            slot->bytes = bytes;
            if (!host_only_) cudaEventCreateWithFlags(&slot->ev, cudaEventDisableTiming);
            pinned_reserved_ += bytes;
            if (pinned_slots_.size() == 1) {  // the first request reserves the double buffer (2 x size)
                PinnedSlot twin{};
                if (!reserve_raw(bytes, &twin.ptr)) return fail("pinned comm slot allocation failed");
                twin.bytes = bytes;
                if (!host_only_) cudaEventCreateWithFlags(&twin.ev, cudaEventDisableTiming);
                pinned_reserved_ += bytes;
                pinned_slots_.push_back(twin);
                slot = &pinned_slots_.front();
            }
        }
        slot->busy = true;
        if (!host_only_ && slot->ev_valid && slot->last_stream != stream) cudaStreamWaitEvent(stream, slot->ev, 0);
        pinned_alloc_ += bytes;
        lv.offset = static_cast<std::int64_t>(slot - pinned_slots_.data());
        return slot->ptr;
    }

    // Consolidation: the open region (slots never handed out yet) first, as the reference fills
    // it; then any fully idle region of the same slot size (recycled); else a new k-slot region.
    void* packed_alloc(std::int64_t bytes, cudaStream_t stream, Live& lv) {
        const std::int64_t k = policy_.consolidate_every_k_mlp;
        Region* reg = nullptr;
        std::size_t slot = 0;
        if (open_ >= 0 && regions_[static_cast<std::size_t>(open_)].slot == bytes &&
            regions_[static_cast<std::size_t>(open_)].handed_out < k) {
            reg = &regions_[static_cast<std::size_t>(open_)];
            slot = static_cast<std::size_t>(reg->handed_out++);
        }
        if (!reg) {
            for (auto& r : regions_) {
                bool idle = r.slot == bytes;
                for (bool u : r.used) idle = idle && !u;
                if (idle && r.handed_out >= k) {
                    reg = &r;
                    r.handed_out = 1;  // the region reopens; slot 0 first, as when it was new
                    slot = 0;
                    break;
                }
            }
        }
        if (!reg) {
            regions_.push_back(Region{});
            reg = &regions_.back();
            if (!reserve_raw(k * bytes, &reg->ptr)) {
                regions_.pop_back();
                return fail("consolidated region allocation failed");
            }
            reg->slot = bytes;
            reg->used.assign(static_cast<std::size_t>(k), false);
            reg->handed_out = 1;
            if (!host_only_) cudaEventCreateWithFlags(&reg->ev, cudaEventDisableTiming);
            packed_reserved_ += k * bytes;
        }
        open_ = reg - regions_.data();
        reg->used[slot] = true;
        if (!host_only_ && reg->ev_valid && reg->last_stream != stream) cudaStreamWaitEvent(stream, reg->ev, 0);
        packed_alloc_ += bytes;
        lv.where = Where::Packed;
        lv.segment = static_cast<std::size_t>(reg - regions_.data());
        lv.offset = static_cast<std::int64_t>(slot);
        return static_cast<char*>(reg->ptr) + static_cast<std::int64_t>(slot) * bytes;
    }

    void record_pinned_release(const Live& lv, cudaStream_t stream) {
        PinnedSlot& s = pinned_slots_[static_cast<std::size_t>(lv.offset)];
        s.busy = false;
        if (!host_only_) {
            cudaEventRecord(s.ev, stream);
            s.ev_valid = true;
            s.last_stream = stream;
        }
    }

    void record_release(const Live& lv, cudaStream_t stream) {
        if (host_only_) return;
        Pending p{lv.segment, lv.offset, lv.offset + lv.bytes, stream, nullptr};
        cudaEventCreateWithFlags(&p.ev, cudaEventDisableTiming);
        cudaEventRecord(p.ev, stream);
        pending_.push_back(p);
    }

    void wait_for_reuse(const Live& lv, cudaStream_t stream) {
        if (host_only_) return;
        for (std::size_t i = 0; i < pending_.size();) {
            Pending& p = pending_[i];
            if (cudaEventQuery(p.ev) == cudaSuccess) {  // retired: forget it
                cudaEventDestroy(p.ev);
                pending_[i] = pending_.back();
                pending_.pop_back();
                continue;
            }
            const bool overlap = p.segment == lv.segment && p.lo < lv.offset + lv.bytes && lv.offset < p.hi;
            if (overlap && p.stream != stream) cudaStreamWaitEvent(stream, p.ev, 0);
            ++i;
        }
    }

    Stats snapshot() {
        std::int64_t cached = 0, frag = 0;
        const std::int64_t threshold = threshold_;  // == trace_.smallest_recurring_request(), kept incrementally
        pool_.free_space(threshold, cached, frag);
        Stats& s = stats_;
        const std::int64_t pinned_res = pinned_reserved_;
        const std::int64_t grad_res = grad_arena_bytes_;
        s.reserved = pool_.reserved() + pinned_res + grad_res + packed_reserved_;
        s.allocated = pool_.allocated() + pinned_alloc_ + grad_alloc_ + packed_alloc_;
        s.free_cached = cached + (pinned_res - pinned_alloc_) + (grad_res - grad_alloc_) +
                        (packed_reserved_ - packed_alloc_);
        s.fragmented = frag;
        s.peak_reserved = std::max(s.peak_reserved, s.reserved);
        s.peak_fragmented = std::max(s.peak_fragmented, s.fragmented);
        s.peak_allocated = std::max(s.peak_allocated, s.allocated);
        return s;
    }

    seqplan::MempoolPolicy policy_;
    seqplan::detail::CachingPool pool_;
    seqplan::Trace trace_;
    std::vector<void*> segments_;
    std::vector<PinnedSlot> pinned_slots_;
    std::vector<Region> regions_;
    std::map<std::int64_t, int> size_seen_;
    std::int64_t threshold_ = 0;
    std::ptrdiff_t open_ = -1;  // the region packed requests currently fill
    std::int64_t packed_reserved_ = 0, packed_alloc_ = 0;
    std::vector<Pending> pending_;
    std::unordered_map<void*, Live> live_;
    std::vector<Stats> per_step_;
    Stats stats_;
    std::string error_;
    void* grad_arena_ = nullptr;
    std::int64_t grad_arena_bytes_ = 0, grad_used_ = 0, grad_alloc_ = 0, grad_live_ = 0;
    std::int64_t pinned_reserved_ = 0, pinned_alloc_ = 0;
    std::int64_t next_id_ = 0;
    std::int64_t host_cursor_ = 0;
    bool host_only_ = false;
};

}  // namespace isp
