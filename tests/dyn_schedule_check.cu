// Host-only check of the power-sum kernel's dynamic-tail schedule
// (csrc/power_sums.cuh: dyn_plan + dyn_chunk): for many (tiles, grid)
// shapes, chunks 0..n_chunks-1 must cover [static_tiles, tiles) exactly once,
// be non-empty, ascend within a chunk, and keep the globally last tile last
// in its chunk (the ragged-tile rule); chunk n_chunks must be empty.
// Built and run by tests/test_dyn_schedule.py.
#include <cstdio>
#include <vector>

#include "../paper_1512_08017_b200/csrc/power_sums.cuh"

static int check(uint64_t tiles, uint64_t grid, uint64_t den, uint64_t chunk, uint64_t max_chunks) {
    const lsq::DynPlan p = lsq::dyn_plan(tiles, grid, den, chunk, max_chunks);
    if (p.n_chunks > max_chunks) return 1;
    std::vector<unsigned char> seen(tiles, 0);
    for (uint64_t c = 0; c < p.n_chunks; ++c) {
        uint64_t first, count;
        lsq::dyn_chunk(c, grid, p.static_tiles, p.s0, p.chunk_min, tiles, first, count);
        if (count == 0) return 2;
        for (uint64_t j = 0; j < count; ++j) {
            const uint64_t t = first + j * grid;
            if (t < p.static_tiles || t >= tiles || seen[t]) return 3;
            seen[t] = 1;
            if (t + 1 == tiles && j + 1 != count) return 4;
        }
    }
    for (uint64_t t = p.static_tiles; t < tiles; ++t)
        if (!seen[t]) return 5;
    uint64_t first, count;
    lsq::dyn_chunk(p.n_chunks, grid, p.static_tiles, p.s0, p.chunk_min, tiles, first, count);
    return count == 0 ? 0 : 6;
}

int main() {
    int cases = 0, bad = 0;
    const uint64_t grids[] = {1, 2, 7, 37, 132, 148, 296};
    const uint64_t shapes[] = {1, 2, 3, 8, 15, 16, 17, 128, 129, 511, 512, 513, 1000, 1884, 7541};
    for (uint64_t g : grids)
        for (uint64_t per : shapes)
            for (uint64_t extra : {uint64_t(0), uint64_t(1), g / 2, g - 1})
                for (uint64_t den : {uint64_t(1), uint64_t(2), uint64_t(4), uint64_t(8)})
                    for (uint64_t chunk : {uint64_t(4), uint64_t(8), uint64_t(16)}) {
                        const uint64_t tiles = per * g + extra;
                        if (tiles < g) continue;
                        const int r = check(tiles, g, den, chunk, 4096);
                        ++cases;
                        if (r) {
                            ++bad;
                            if (bad < 10)
                                std::printf("FAIL code %d tiles=%llu grid=%llu den=%llu chunk=%llu\n", r,
                                            (unsigned long long)tiles, (unsigned long long)g,
                                            (unsigned long long)den, (unsigned long long)chunk);
                        }
                    }
    // the bench shape: n = 4e9 points of 3584-point tiles over 148 CTAs, and a
    // tiny record cap (forces the chunk floor to double)
    ++cases;
    if (check((4000000000ull + 3583) / 3584, 148, 2, 8, 4096)) ++bad;
    ++cases;
    if (check(1116072, 148, 2, 8, 300)) ++bad;
    std::printf("%d cases, %d failed\n", cases, bad);
    return bad ? 1 : 0;
}
