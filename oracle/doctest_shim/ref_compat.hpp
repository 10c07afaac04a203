// Force-included (-include) when compiling the reference's own unit tests.
// The shipped header declares `friend bool operator==(const PreparedLayer&,
// const PreparedLayer&) = default;` (pipeline.hpp:64) but QuantSpec
// (quant.hpp:15-20) has no operator==, so with g++ 13 the defaulted
// comparison is deleted and test_pipeline.cpp:108 does not compile.  This
// supplies the obvious member-wise comparison before pipeline.hpp is seen.
// TEST INFRASTRUCTURE ONLY.
#pragma once
#include "convrot/quant.hpp"
namespace convrot {
inline bool operator==(const QuantSpec& a, const QuantSpec& b) {
  return a.bits == b.bits && a.granularity == b.granularity;
}
}  // namespace convrot
