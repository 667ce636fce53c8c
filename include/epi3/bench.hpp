#pragma once
// Forwarding header: the reference include path (include/epi3/bench.hpp) -> the drop-in API.
#include "epi3/api.hpp"
