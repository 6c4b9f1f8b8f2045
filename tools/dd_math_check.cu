// Host build of csrc/dd_math.cuh for CPU checks (tests/test_dd_math.py):
//   dd_math_check <in.f64> <out.f64>   -> atan_cr(x_i), asinh_cr(x_i), pow25_cr(|x_i|) interleaved
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#include "../paper_2602_12242_b200/csrc/dd_math.cuh"

int main(int argc, char** argv) {
    if (argc != 3) return 2;
    FILE* f = fopen(argv[1], "rb");
    if (!f) return 3;
    std::vector<double> x;
    double v;
    while (fread(&v, sizeof v, 1, f) == 1) x.push_back(v);
    fclose(f);
    std::vector<double> out(3 * x.size());
    for (size_t i = 0; i < x.size(); ++i) {
        out[3 * i] = ddm::atan_cr(x[i]);
        out[3 * i + 1] = ddm::asinh_cr(x[i]);
        out[3 * i + 2] = ddm::pow25_cr(fabs(x[i]));
    }
    f = fopen(argv[2], "wb");
    if (!f) return 4;
    fwrite(out.data(), sizeof(double), out.size(), f);
    fclose(f);
    return 0;
}
