// Loads a measured VPro CSV (tools/nvlink_kernels.py --vpro) with the reference API
// (load_bandwidth_csv_file, bandwidth.hpp:214-253) and prints, per op and measured size, the
// looked-up bandwidth and the one at the geometric midpoint to the next size (log-log
// interpolation, bandwidth.hpp:166-196), plus collective_time for the 7B-32K p-rank block.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "seqplan/bandwidth.hpp"

using namespace seqplan;

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const BandwidthProfile prof = load_bandwidth_csv_file(argv[1]);
    std::printf("[");
    bool first = true;
    for (const auto& e : prof.entries()) {
        if (e.axis != MeshAxis::Intra) continue;
        const double at = prof.lookup(e.op, e.participants, MeshAxis::Intra, e.message_bytes);
        const std::int64_t mid = static_cast<std::int64_t>(double(e.message_bytes) * 2.0);
        const double at_mid = prof.lookup(e.op, e.participants, MeshAxis::Intra, mid);
        const double t = collective_time(prof, e.op, e.message_bytes, e.participants, MeshAxis::Inter);
        std::printf("%s{\"op\":\"%s\",\"p\":%lld,\"v\":%lld,\"bw\":%.9g,\"lookup\":%.9g,\"lookup_2v\":%.9g,\"tau\":%.9g}",
                    first ? "" : ",", to_string(e.op), (long long)e.participants, (long long)e.message_bytes,
                    e.bandwidth, at, at_mid, t);
        first = false;
    }
    std::printf("]\n");
    return 0;
}
