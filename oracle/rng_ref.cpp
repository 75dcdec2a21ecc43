// Test infrastructure only: prints libstdc++'s own std::mt19937_64 and
// std::normal_distribution<double>(0,1) draws, the generators the reference uses
// for cold starts and basis growth (spectral.hpp:135-139, pipeline.hpp:104-107),
// so the oracle's pure-Python restatement can be pinned to them.
// usage: rng_ref <seed> <count>
#include <cstdio>
#include <cstdlib>
#include <random>
int main(int argc, char** argv) {
    unsigned long long seed = argc > 1 ? std::strtoull(argv[1], nullptr, 0) : 1;
    int count = argc > 2 ? std::atoi(argv[2]) : 8;
    std::mt19937_64 raw(seed);
    for (int i = 0; i < count; ++i) std::printf("u %llu\n", (unsigned long long)raw());
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (int i = 0; i < count; ++i) std::printf("g %a\n", gauss(rng));
    return 0;
}
