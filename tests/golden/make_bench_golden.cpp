// Generates tests/golden/bench_golden.json from the UNMODIFIED reference driver.hpp / oracle.hpp (build container only):
//   g++ -std=c++20 -O2 -pthread -I/root/reference/proj/include tests/golden/make_bench_golden.cpp -o /tmp/mbg && /tmp/mbg > tests/golden/bench_golden.json
// benchmark() reports (driver.hpp:253-302) with the three timing columns blanked, and the two exact solvers
// (oracle.hpp:45-149) on generated instances.
#include <iostream>
#include <sstream>
#include <projmotif/driver.hpp>
#include <projmotif/oracle.hpp>
#include <projmotif/planted.hpp>

using namespace projmotif;

static std::string blank_timings(const std::string& tsv) {
    std::istringstream in(tsv);
    std::string line, out;
    bool first = true;
    while (std::getline(in, line)) {
        if (first) {
            out += line + "\n";
            first = false;
            continue;
        }
        std::vector<std::string> cols;
        std::istringstream ls(line);
        std::string col;
        while (std::getline(ls, col, '\t')) cols.push_back(col);
        for (std::size_t i = 6; i < cols.size(); ++i) cols[i] = "-";
        for (std::size_t i = 0; i < cols.size(); ++i) out += cols[i] + (i + 1 < cols.size() ? "\t" : "\n");
    }
    return out;
}

static std::string quote(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '\n') o += "\\n";
        else if (c == '\t') o += "\\t";
        else o += c;
    }
    return o + "\"";
}

int main() {
    std::cout << "{\n  \"bench\": [\n";
    struct Cfg { int instances, t, n, l, d; std::uint64_t seed; int s; long m; };
    const Cfg cfgs[] = {{20, 3, 10, 3, 1, 1, 3, 0}, {8, 4, 14, 5, 1, 7, 2, 6}, {5, 5, 20, 6, 2, 11, 2, 0}};
    for (std::size_t c = 0; c < 3; ++c) {
        BenchConfig b;
        b.instances = cfgs[c].instances; b.t = cfgs[c].t; b.n = cfgs[c].n; b.l = cfgs[c].l; b.d = cfgs[c].d; b.seed = cfgs[c].seed;
        b.run.s = cfgs[c].s;
        if (cfgs[c].m > 0) b.run.m = cfgs[c].m;
        std::cout << "    {\"instances\": " << b.instances << ", \"t\": " << b.t << ", \"n\": " << b.n << ", \"l\": " << b.l
                  << ", \"d\": " << b.d << ", \"seed\": " << b.seed << ", \"s\": " << cfgs[c].s << ", \"m\": " << cfgs[c].m
                  << ", \"tsv\": " << quote(blank_timings(benchmark(b))) << "}" << (c + 1 < 3 ? "," : "") << "\n";
    }
    std::cout << "  ],\n  \"oracle\": [\n";
    struct Inst { int t, n, l, d; std::uint64_t seed; };
    const Inst insts[] = {{3, 70, 8, 1, 5}, {4, 30, 6, 1, 9}, {6, 40, 9, 2, 3}, {20, 100, 10, 2, 42}};
    for (std::size_t i = 0; i < 4; ++i) {
        const PlantedInstance inst = generate_planted(insts[i].t, insts[i].n, insts[i].l, insts[i].d, insts[i].seed);
        const MedianStringResult med = median_string(inst.sequences, insts[i].l);
        std::cout << "    {\"t\": " << insts[i].t << ", \"n\": " << insts[i].n << ", \"l\": " << insts[i].l << ", \"d\": " << insts[i].d
                  << ", \"seed\": " << insts[i].seed << ", \"median\": " << quote(med.median) << ", \"total_distance\": " << med.total_distance;
        if (i < 2) {
            const NaiveMfpResult nv = naive_mfp(inst.sequences, insts[i].l);
            std::cout << ", \"naive_score\": " << nv.score << ", \"naive_consensus\": " << quote(nv.consensus) << ", \"naive_positions\": [";
            for (std::size_t k = 0; k < nv.positions.size(); ++k) std::cout << nv.positions[k] << (k + 1 < nv.positions.size() ? ", " : "");
            std::cout << "]";
        }
        std::cout << "}" << (i + 1 < 4 ? "," : "") << "\n";
    }
    std::cout << "  ]\n}\n";
    return 0;
}
