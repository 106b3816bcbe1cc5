// seqplan/placement.hpp — rank nesting of the process groups.
//
// Restates proj/include/seqplan/placement.hpp:12-59. Ranks are nested tp/sp
// innermost (stride 1), then ps (stride max(tp,sp)), then oss (stride act*ps);
// a group of size g and stride t spans t*g consecutive ranks and is intra when
// that span fits a node, mixed when it straddles nodes with stride < node
// size, inter otherwise. Note: for the single-box ISP plan
// sp = ps = p the ps group classifies as inter even though every rank is on
// the same NVSwitch; the output is kept bit-exact and the executor uses the
// physical layout (all p GPUs of one box, uniform peer bandwidth).
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>

#include "seqplan/bandwidth.hpp"
#include "seqplan/strategy.hpp"

namespace seqplan {

enum class GroupKind { TpSp, Ps, Oss, Gs, Dp };

inline const char* to_string(GroupKind k) {
    static const char* const names[] = {"tp/sp", "ps", "oss", "gs", "dp"};
    const int i = static_cast<int>(k);
    return (i >= 0 && i < 5) ? names[i] : "?";
}

struct MeshPlacement {
    std::map<GroupKind, MeshAxis> axis;
    MeshAxis operator[](GroupKind k) const { return axis.at(k); }
};

inline MeshPlacement place_groups(const ClusterConfig& cluster, const Strategy& s) {
    const std::int64_t node = cluster.gpus_per_node;
    auto axis_of = [node](std::int64_t stride, std::int64_t size) -> MeshAxis {
        if (size <= 1 || stride * size <= node) return MeshAxis::Intra;
        return stride < node ? MeshAxis::Mixed : MeshAxis::Inter;
    };
    const std::int64_t inner = std::max(s.tp, s.sp);
    const std::int64_t sync_group = cluster.total_gpus / (s.pp * s.tp * s.ps);
    MeshPlacement m;
    m.axis[GroupKind::TpSp] = axis_of(1, inner);
    m.axis[GroupKind::Ps] = axis_of(inner, s.ps);
    m.axis[GroupKind::Oss] = axis_of(inner * s.ps, s.oss);
    m.axis[GroupKind::Gs] = axis_of(inner * s.ps, sync_group);
    m.axis[GroupKind::Dp] = axis_of(s.sp, s.dp);
    return m;
}

}  // namespace seqplan
