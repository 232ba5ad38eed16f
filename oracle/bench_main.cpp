// oracle/bench_main.cpp — TEST/MEASUREMENT INFRASTRUCTURE ONLY.
// A main() for the reference's own benchmark harness, lsqfit::run_benchmark
// (proj/include/lsqfit/bench.hpp:26-27, proj/src/bench.cpp), which the
// reference's CLI exposes as `lsqfit bench --points N --degree M --chunks C
// --repeat R --seed S` (cli.cpp; target command in proj/tools/CMakeLists.txt:6-10).
// The CLI itself cannot be built here (CLI11 is not vendored), so this file
// stands in for it. Built twice by oracle/Makefile: against the reference's
// own sources (bench_on_ref) and against the B200 drop-in (bench_on_b200).
#include <cstdio>
#include <cstdlib>

#include "lsqfit/bench.hpp"

int main(int argc, char** argv) {
    const std::size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 10000000ull;
    const int degree = argc > 2 ? std::atoi(argv[2]) : 4;
    const int chunks = argc > 3 ? std::atoi(argv[3]) : 8;
    const int reps = argc > 4 ? std::atoi(argv[4]) : 5;
    const unsigned long long seed = argc > 5 ? std::strtoull(argv[5], nullptr, 10) : 1ull;
    const lsqfit::BenchReport r = lsqfit::run_benchmark(n, degree, chunks, reps, seed);
    std::printf(
        "{\"n_points\": %zu, \"degree\": %d, \"chunks\": %d, \"repetitions\": %d, "
        "\"sequential_median_s\": %.9g, \"sequential_min_s\": %.9g, \"parallel_median_s\": %.9g, "
        "\"parallel_min_s\": %.9g, \"speedup\": %.6g, \"max_relative_deviation\": %.6g, \"valid\": %s}\n",
        r.n_points, r.degree, r.chunks, r.repetitions, r.sequential_median_s, r.sequential_min_s,
        r.parallel_median_s, r.parallel_min_s, r.speedup, r.max_relative_deviation, r.valid ? "true" : "false");
    return r.valid ? 0 : 1;
}
