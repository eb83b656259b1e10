// Exercises include/xband_b200.hpp the way a reference caller would
// (pipeline.cpp:99-137 loop swapped for one extend_batch call).
// argv[1] == "gpu": also run extensions and check the Appendix-B KATs.
#include <cstdio>
#include <cstring>
#include <vector>

#include "xband_b200.hpp"

using namespace xband_b200;

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    auto s = ScoringScheme::match_mismatch(1, -1, -1, 5);
    if (s.sim('A', 'A') != 1 || s.sim('N', 'N') != -1) return 10;
    SequencePool pool(s);
    pool.add("AAAAAAAAAA");
    pool.add("AAAAAAAAAA");
    try {
        std::vector<SeedAlignment> done;
        std::vector<FailedUnit> failed;
        extend_batch(pool, {ExtensionTask{0, 0, 7, 0, 0}}, 2, 8, done, failed);
        return 11;  // must have thrown
    } catch (const DanglingReference&) {
    }
    try {
        extend_seed(pool, ExtensionTask{0, 0, 1, 9, 0}, 4, 16);
        return 12;
    } catch (const SeedOutOfBounds&) {
    }
    if (!gpu) {
        std::puts("shim cpu ok");
        return 0;
    }
    // test_align.cpp:243-256: 3 + 4 + 3 = 10
    SeedAlignment a = extend_seed(pool, ExtensionTask{0, 0, 1, 3, 3}, 4, 16);
    if (a.seed_score != 4 || a.left.score != 3 || a.right.score != 3 || a.total != 10) return 13;
    // band failure names its side
    SequencePool p2(s);
    p2.add("AAAAAAAAAAAAAAAAAAAAAAAAAAAAAAAA");
    p2.add("AAAATAAAATAAAATAAAATAAAATAAAATAA");
    try {
        extend_seed(p2, ExtensionTask{0, 0, 1, 0, 0}, 0, 1);
        return 14;
    } catch (const BandExceededError& e) {
        if (e.side != 'R' || e.observed_spread <= 1) return 15;
    }
    std::puts("shim gpu ok");
    return 0;
}
