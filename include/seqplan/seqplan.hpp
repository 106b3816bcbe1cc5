// seqplan/seqplan.hpp — umbrella header of the hot-path subset.
//
// Mirrors proj/include/seqplan/seqplan.hpp:3-12 for the headers the ISP
// executor owns. The planner front-end (config.hpp, report.hpp, search.hpp) is
// out of scope and intentionally absent.
#pragma once

#include "seqplan/bandwidth.hpp"
#include "seqplan/cost.hpp"
#include "seqplan/mempool.hpp"
#include "seqplan/model.hpp"
#include "seqplan/overlap_sim.hpp"
#include "seqplan/placement.hpp"
#include "seqplan/strategy.hpp"
