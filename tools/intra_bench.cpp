// Host intra-payload parse micro-benchmark (first I-frame of a stream):
// sequential tree walk, parallel tree walk, value symbols, full parse_intra;
// optionally N concurrent parse_intra calls (as the decoder runs them).
//   g++ -O3 -std=c++17 -I include tools/intra_bench.cpp -o tools/intra_bench.bin -lpthread
//   tools/intra_bench.bin tests/golden/streams/cfg3_Y.hivc [concurrent]
#include "../paper_2008_10273_b200/csrc/parse.cpp"

#include <chrono>
#include <fstream>
#include <iterator>

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
    const int conc = argc > 2 ? std::atoi(argv[2]) : 0;
    StreamHeader hd = parse_header(d.data(), d.size());
    std::vector<std::pair<size_t, size_t>> gops;
    split_gops(d.data(), d.size(), hd, gops);
    const uint8_t* p = d.data() + gops[0].first;
    uint32_t plen;
    std::memcpy(&plen, p + 3, 4);
    const uint8_t* pd = p + 7;
    uint32_t nbits;
    intra_tree_span(pd, plen, 0, nbits);
    std::vector<uint64_t> bits;
    const int reps = 10;
    double t0 = now();
    for (int r = 0; r < reps; ++r) intra_tree_seq(pd, 0, nbits, hd.height, hd.width, bits);
    const double ts = (now() - t0) / reps;
    t0 = now();
    std::vector<uint64_t> local;
    for (int r = 0; r < reps; ++r) intra_tree_par(pd, 0, nbits, hd.height, hd.width, 4, bits, local);
    const double tp = (now() - t0) / reps;
    std::vector<int32_t> idx;
    t0 = now();
    for (int r = 0; r < reps; ++r) intra_symbols(pd, plen, 4 + (nbits + 7) / 8, idx);
    const double tv = (now() - t0) / reps;
    IntraJob job;
    t0 = now();
    for (int r = 0; r < reps; ++r) parse_intra(pd, plen, 0, hd.height, hd.width, 1, hd.intra_levels, job, bits);
    const double ti = (now() - t0) / reps;
    std::printf("tree seq %.0f us | tree par4 %.0f us | values %.0f us | parse_intra %.0f us\n", ts * 1e6, tp * 1e6,
                tv * 1e6, ti * 1e6);
    if (conc > 0) {  // warm scratch per thread (as the decoder keeps it per slot), then time
        std::vector<IntraJob> jobs(conc);
        std::vector<std::vector<uint64_t>> bs(conc);
        for (int round = 0; round < 3; ++round) {
            t0 = now();
            std::vector<std::thread> th;
            for (int c = 0; c < conc; ++c)
                th.emplace_back([&, c]() {
                    parse_intra(pd, plen, 0, hd.height, hd.width, 1, hd.intra_levels, jobs[c], bs[c]);
                });
            for (auto& t : th) t.join();
            std::printf("%d concurrent parse_intra (round %d): %.0f us\n", conc, round, (now() - t0) * 1e6);
        }
    }
    return 0;
}
