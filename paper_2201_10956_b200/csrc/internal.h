// internal.h — shared by host.cpp and engine.cu (not part of the ABI).
#pragma once
#include <cstdint>
#include <string>

namespace e3 {
// Records the thread-local message returned by e3_last_error() and passes
// the status through.
int fail(int code, const std::string& msg);
uint64_t triple_rank(uint64_t M, uint64_t i0, uint64_t i1, uint64_t i2);
void triple_unrank(uint64_t M, uint64_t r, uint32_t* t);
}  // namespace e3
