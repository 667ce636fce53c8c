// Forwarding header: the reference include path epi3/common.hpp maps to the
// single drop-in surface of the B200 engine.
#pragma once
#include "epi3/api.hpp"
