// TEST INFRASTRUCTURE: a C-ABI shim around the REFERENCE's own keyed RNG
// (proj/src/core/rng.hpp, header-only, compiled straight from /root/reference
// by oracle/Makefile into oracle/_ref/libref_rng.so). tests/test_ref_rng.py
// checks the oracle restatement (cpkit_oracle.cpp) against it bit for bit, and
// tests/golden/ref_rng.json holds vectors made from it (make_ref_rng_golden.py)
// so the check also runs where /root/reference is absent.
#include <cstdint>

#include "rng.hpp"  // -I /root/reference/proj/src/core

extern "C" {
double ref_uniform(std::uint64_t seed, std::uint64_t stream, std::uint64_t index, double a, double b) {
    return cpkit::rng::uniform(seed, stream, index, a, b);
}
double ref_gaussian(std::uint64_t seed, std::uint64_t stream, std::uint64_t index) {
    return cpkit::rng::gaussian(seed, stream, index);
}
std::uint64_t ref_mix64(std::uint64_t x) { return cpkit::rng::mix64(x); }
std::uint64_t ref_derive(std::uint64_t h, std::uint64_t v) { return cpkit::rng::derive(h, v); }
std::uint64_t ref_keyed(std::uint64_t seed, std::uint64_t stream, std::uint64_t index, std::uint64_t salt) {
    return cpkit::rng::keyed(seed, stream, index, salt);
}
}
