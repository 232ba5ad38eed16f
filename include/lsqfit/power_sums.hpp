// lsqfit/power_sums.hpp — the hot path's API (reference
// proj/include/lsqfit/power_sums.hpp:13-31), implemented on the B200 by one
// fused streaming kernel (paper_1512_08017_b200/csrc/power_sums.cuh).
#pragma once

#include <cstddef>
#include <vector>

#include "lsqfit/dataset.hpp"

namespace lsqfit {

// s[k] = sum x^k (k = 0..2m), t[j] = sum x^j y (j = 0..m); s[0] == n exactly.
struct PowerSums {
    int degree = 0;
    std::vector<double> s;
    std::vector<double> t;
    std::size_t n = 0;
};

// One pass over the dataset. std::invalid_argument for degree < 0; any
// degree >= 0 is accepted, as in the reference (degrees up to 12 run the fused
// kernel, larger ones the any-degree kernel); OverflowError when a sum is
// non-finite.
PowerSums accumulate(const Dataset& dataset, int degree);

// Same contract with a caller-chosen chunk count (std::invalid_argument for
// chunks < 1). The GPU grid is the parallelism; the result is a pure function
// of (dataset, degree, chunks) and chunks == 1 is bit-identical to accumulate().
PowerSums accumulate_parallel(const Dataset& dataset, int degree, int chunks);

}  // namespace lsqfit
