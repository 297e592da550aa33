// spikecam/metrics.hpp -- the reference's header name (proj/include/spikecam/metrics.hpp)
// for callers of the C++ drop-in: the whole surface is declared in
// spikecam/b200.hpp and implemented over the sm_100a C-ABI.
#pragma once
#include "spikecam/b200.hpp"
