// Host build of csrc/glibc_exp.cuh for tests/test_host.py: reads float64 arguments from argv[1],
// writes kt::glibc_exp of each to argv[2].  Built with g++ -ffp-contract=off.
#include <cstdio>
#include <vector>

#include "glibc_exp.cuh"

int main(int argc, char** argv) {
    if (argc != 3) return 2;
    FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 3;
    std::vector<double> x;
    double v;
    while (std::fread(&v, 8, 1, f) == 1) x.push_back(v);
    std::fclose(f);
    for (double& a : x) a = kt::glibc_exp(a, kt::kExpTable);
    FILE* g = std::fopen(argv[2], "wb");
    if (!g) return 4;
    std::fwrite(x.data(), 8, x.size(), g);
    std::fclose(g);
    return 0;
}
