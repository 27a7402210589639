// Host parser micro-benchmark: time parse_intra / parse_flow / parse_residual
// on the frame records of one GOP of a stream.
//   g++ -O3 -std=c++17 -I include tools/parse_bench.cpp paper_2008_10273_b200/csrc/parse.cpp -o /tmp/pb
//   /tmp/pb tests/golden/streams/cfg3_Y.hivc
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <vector>

#include "../paper_2008_10273_b200/csrc/parse.h"

namespace hivc {
void set_last_error(const std::string&) {}
}  // namespace hivc

using namespace hivc;

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
    std::ifstream f(argv[1], std::ios::binary);
    std::vector<uint8_t> d((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    StreamHeader hd = parse_header(d.data(), d.size());
    std::vector<std::pair<size_t, size_t>> gops;
    split_gops(d.data(), d.size(), hd, gops);
    const uint8_t* p = d.data() + gops[0].first;
    uint16_t nf;
    std::memcpy(&nf, p, 2);
    size_t pos = 2;
    double t_intra = 0, t_flow = 0, t_res = 0;
    int n_intra = 0, n_flow = 0, n_res = 0;
    const int reps = 20;
    IntraJob ij;
    FlowJob fj;
    ResidualJob rj;
    std::vector<uint64_t> bits;
    for (int fi = 0; fi < nf; ++fi) {
        uint8_t ft = p[pos];
        uint32_t plen;
        std::memcpy(&plen, p + pos + 1, 4);
        pos += 5;
        const uint8_t* pd = p + pos;
        pos += plen;
        double t0 = now();
        for (int r = 0; r < reps; ++r) {
            if (ft == 0)
                parse_intra(pd, plen, 0, hd.height, hd.width, hd.channels, hd.intra_levels, ij, bits);
            else
                parse_flow(pd, plen, 0, hd.height, hd.width, hd.flow_levels, fj);
        }
        double dt = (now() - t0) / reps;
        if (ft == 0) t_intra += dt, ++n_intra;
        else t_flow += dt, ++n_flow;
        uint32_t rlen;
        std::memcpy(&rlen, p + pos, 4);
        pos += 4;
        t0 = now();
        for (int r = 0; r < reps; ++r) parse_residual(p + pos, rlen, 0, hd.height, hd.width, hd.channels, rj);
        t_res += (now() - t0) / reps;
        ++n_res;
        pos += rlen;
    }
    std::printf("intra %.1f us/frame (%d) | flow %.1f us/frame (%d) | residual %.1f us/frame (%d)\n",
                1e6 * t_intra / std::max(1, n_intra), n_intra, 1e6 * t_flow / std::max(1, n_flow), n_flow,
                1e6 * t_res / std::max(1, n_res), n_res);
    return 0;
}
