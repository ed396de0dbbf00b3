// projmotif_b200 — command-line front end of the B200 PROJECTION path, mirroring the reference's
// `projmotif find`, `gen`, `oracle` and `bench` (tools/projmotif.cpp:67-148, 164-211): same flags, same
// JSON/TSV reports (report.hpp schema v1), same exit codes (0 ok, 2 parameter/usage, 3 no enriched bucket,
// 4 parse/I-O).  `oracle --method median` runs on the device; `--method naive` is the exponential host solver.
//
//   g++ -std=c++17 -O2 -Iinclude tools/projmotif_b200.cpp -Lpaper_1605_06904_b200 -lpm_b200 \
//       -Wl,-rpath,$PWD/paper_1605_06904_b200 -o projmotif_b200
#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "projmotif_b200.hpp"

namespace pmx = projmotif_b200;

namespace {

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

int env_workers() {  // tools/projmotif.cpp:17-26
    if (const char* env = std::getenv("PROJMOTIF_WORKERS")) {
        char* end = nullptr;
        const long v = std::strtol(env, &end, 10);
        if (end != env && *end == '\0' && v >= 1 && v <= 4096) return static_cast<int>(v);
    }
    return 1;
}

pmx::SequenceSet read_input(const std::string& path) {
    std::ostringstream buffer;
    if (path == "-") {
        buffer << std::cin.rdbuf();
    } else {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw pmx::IoError("cannot open input file: " + path);
        buffer << in.rdbuf();
    }
    return pmx::parse_fasta(buffer.str());
}

void write_file(const std::string& path, const std::string& content) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw pmx::IoError("cannot open output file: " + path);
    out << content;
    out.flush();
    if (!out) throw pmx::IoError("failed writing to: " + path);
}

// "--name value" / "--name=value" / bare flags
struct Args {
    std::map<std::string, std::string> values;
    std::map<std::string, bool> flags;
};

Args parse_flags(int argc, char** argv, int first, const std::vector<std::string>& options,
                 const std::vector<std::string>& flags, const std::map<std::string, std::string>& aliases) {
    Args out;
    for (int i = first; i < argc; ++i) {
        std::string arg = argv[i], value;
        bool has_value = false;
        const std::size_t eq = arg.find('=');
        if (arg.rfind("--", 0) == 0 && eq != std::string::npos) {
            value = arg.substr(eq + 1);
            arg = arg.substr(0, eq);
            has_value = true;
        }
        if (aliases.count(arg)) arg = aliases.at(arg);
        if (std::find(flags.begin(), flags.end(), arg) != flags.end()) {
            out.flags[arg] = true;
            continue;
        }
        if (std::find(options.begin(), options.end(), arg) == options.end()) {
            throw UsageError("The following argument was not expected: " + arg);
        }
        if (!has_value) {
            if (i + 1 >= argc) throw UsageError(arg + ": 1 required TEXT missing");
            value = argv[++i];
        }
        out.values[arg] = value;
    }
    return out;
}

template <typename T>
T to_number(const std::string& name, const std::string& text) {
    std::size_t used = 0;
    T v{};
    try {
        if constexpr (std::is_same_v<T, double>) {
            v = std::stod(text, &used);
        } else if constexpr (std::is_same_v<T, std::uint64_t>) {
            if (!text.empty() && text[0] == '-') throw std::invalid_argument("negative");
            v = std::stoull(text, &used);
        } else {
            v = static_cast<T>(std::stoll(text, &used));
        }
    } catch (const std::exception&) {
        throw UsageError("Could not convert: " + name + " = " + text);
    }
    if (used != text.size()) throw UsageError("Could not convert: " + name + " = " + text);
    return v;
}

template <typename T>
std::optional<T> opt_number(const Args& a, const std::string& name) {
    const auto it = a.values.find(name);
    if (it == a.values.end()) return std::nullopt;
    return to_number<T>(name, it->second);
}

template <typename T>
T required(const Args& a, const std::string& name) {
    const auto v = opt_number<T>(a, name);
    if (!v) throw UsageError(name + " is required");
    return *v;
}

int usage(std::ostream& os) {
    os << "planted (l,d)-motif discovery by random projection (B200 path)\n"
          "Usage: projmotif_b200 find -i FASTA --l L --d D [--k K] [--s S] [--m M] [--q Q] [--seed N] [--workers N]\n"
          "                           [--backend dense|grouped|auto] [--max-em-iters N] [--s-floor N] [--no-early-stop]\n"
          "                           [--format json|tsv] [--device N]\n"
          "       projmotif_b200 gen --t T --n N --l L --d D [--seed N] -o OUT.fasta\n"
          "       projmotif_b200 oracle -i FASTA --l L [--method naive|median] [--limit N]\n"
          "       projmotif_b200 bench [--instances N] [--t T] [--n N] [--l L] [--d D] [--seed N] [--s S] [--m M] [--q Q]\n"
          "                            [--workers N] [--backend dense|grouped|auto] [--naive-limit N] [--median-limit N]\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "A subcommand is required\n";
        usage(std::cerr);
        return 2;
    }
    const std::string cmd = argv[1];
    if (cmd == "-h" || cmd == "--help") return usage(std::cout);
    try {
        if (cmd == "find") {
            const Args a = parse_flags(argc, argv, 2,
                                       {"--input", "--l", "--d", "--k", "--s", "--m", "--q", "--seed", "--workers", "--backend",
                                        "--max-em-iters", "--s-floor", "--format", "--device"},
                                       {"--no-early-stop"}, {{"-i", "--input"}});
            if (!a.values.count("--input")) throw UsageError("--input is required");
            const std::string backend = a.values.count("--backend") ? a.values.at("--backend") : "auto";
            if (backend != "dense" && backend != "grouped" && backend != "auto") throw UsageError("--backend: " + backend + " not in {dense,grouped,auto}");
            const std::string format = a.values.count("--format") ? a.values.at("--format") : "json";
            if (format != "json" && format != "tsv") throw UsageError("--format: " + format + " not in {json,tsv}");
            pmx::RunConfig config;
            config.l = required<int>(a, "--l");
            config.d = required<int>(a, "--d");
            config.k = opt_number<int>(a, "--k");
            config.s = opt_number<int>(a, "--s");
            config.m = opt_number<std::int64_t>(a, "--m");
            config.q = opt_number<double>(a, "--q").value_or(0.95);
            config.seed = opt_number<std::uint64_t>(a, "--seed").value_or(0);
            config.workers = opt_number<int>(a, "--workers").value_or(env_workers());
            config.backend = backend == "dense" ? pmx::HashBackend::dense : backend == "grouped" ? pmx::HashBackend::grouped : pmx::HashBackend::automatic;
            config.max_em_iters = opt_number<int>(a, "--max-em-iters").value_or(5);
            config.s_floor = opt_number<int>(a, "--s-floor").value_or(3);
            config.early_stop = !a.flags.count("--no-early-stop");
            if (const auto dev = opt_number<int>(a, "--device")) pmx::Device::instance().set_device(*dev);
            const pmx::SequenceSet seqs = read_input(a.values.at("--input"));
            const pmx::RunResult result = pmx::run(config, seqs);
            std::cout << (format == "tsv" ? pmx::render_result_tsv(result) : pmx::render_result_json(result));
        } else if (cmd == "gen") {
            const Args a = parse_flags(argc, argv, 2, {"--t", "--n", "--l", "--d", "--seed", "--out"}, {}, {{"-o", "--out"}});
            if (!a.values.count("--out")) throw UsageError("--out is required");
            const pmx::PlantedInstance inst =
                pmx::generate_planted(required<int>(a, "--t"), required<int>(a, "--n"), required<int>(a, "--l"),
                                      required<int>(a, "--d"), opt_number<std::uint64_t>(a, "--seed").value_or(1));
            const std::string out = a.values.at("--out");
            write_file(out, pmx::serialize_fasta(inst.sequences));
            write_file(out + ".truth.json", pmx::truth_json(inst));
            std::cerr << "wrote " << out << " and " << out << ".truth.json\n";
        } else if (cmd == "oracle") {  // tools/projmotif.cpp:115-125, 187-204
            const Args a = parse_flags(argc, argv, 2, {"--input", "--l", "--method", "--limit", "--device"}, {}, {{"-i", "--input"}});
            if (!a.values.count("--input")) throw UsageError("--input is required");
            const std::string method = a.values.count("--method") ? a.values.at("--method") : "naive";
            if (method != "naive" && method != "median") throw UsageError("--method: " + method + " not in {naive,median}");
            const int l = required<int>(a, "--l");
            const auto limit = opt_number<std::uint64_t>(a, "--limit");
            if (const auto dev = opt_number<int>(a, "--device")) pmx::Device::instance().set_device(*dev);
            const pmx::SequenceSet seqs = read_input(a.values.at("--input"));
            std::string doc = "{\n";
            if (method == "naive") {
                const pmx::NaiveMfpResult res = pmx::naive_mfp(seqs, l, limit.value_or(100000000ULL));
                doc += "  \"method\": \"naive\",\n  \"score\": " + std::to_string(res.score) + ",\n  \"positions\": " +
                       pmx::detail::json_int_array(res.positions, "  ") + ",\n  \"consensus\": " + pmx::detail::json_string(res.consensus) + "\n";
            } else {
                const pmx::MedianStringResult res = pmx::median_string(seqs, l, limit.value_or(16777216ULL));
                doc += "  \"method\": \"median\",\n  \"median\": " + pmx::detail::json_string(res.median) +
                       ",\n  \"total_distance\": " + std::to_string(res.total_distance) + "\n";
            }
            std::cout << doc << "}\n";
        } else if (cmd == "bench") {  // tools/projmotif.cpp:127-148, 205-210
            const Args a = parse_flags(argc, argv, 2,
                                       {"--instances", "--t", "--n", "--l", "--d", "--seed", "--s", "--m", "--q", "--workers",
                                        "--backend", "--naive-limit", "--median-limit", "--device"},
                                       {}, {});
            pmx::BenchConfig bench;
            bench.instances = opt_number<int>(a, "--instances").value_or(bench.instances);
            bench.t = opt_number<int>(a, "--t").value_or(bench.t);
            bench.n = opt_number<int>(a, "--n").value_or(bench.n);
            bench.l = opt_number<int>(a, "--l").value_or(bench.l);
            bench.d = opt_number<int>(a, "--d").value_or(bench.d);
            bench.seed = opt_number<std::uint64_t>(a, "--seed").value_or(bench.seed);
            bench.run.s = opt_number<int>(a, "--s").value_or(3);  // the derived threshold is unattainable at oracle scale
            bench.run.m = opt_number<std::int64_t>(a, "--m");
            bench.run.q = opt_number<double>(a, "--q").value_or(bench.run.q);
            bench.run.workers = opt_number<int>(a, "--workers").value_or(env_workers());
            const std::string backend = a.values.count("--backend") ? a.values.at("--backend") : "auto";
            if (backend != "dense" && backend != "grouped" && backend != "auto") throw UsageError("--backend: " + backend + " not in {dense,grouped,auto}");
            bench.run.backend = backend == "dense" ? pmx::HashBackend::dense : backend == "grouped" ? pmx::HashBackend::grouped : pmx::HashBackend::automatic;
            bench.naive_limit = opt_number<std::uint64_t>(a, "--naive-limit").value_or(bench.naive_limit);
            bench.median_limit = opt_number<std::uint64_t>(a, "--median-limit").value_or(bench.median_limit);
            if (const auto dev = opt_number<int>(a, "--device")) pmx::Device::instance().set_device(*dev);
            std::cout << pmx::benchmark(bench);
        } else {
            throw UsageError("unknown subcommand: " + cmd + " (find, gen, oracle, bench)");
        }
        return 0;
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return 2;
    } catch (const pmx::NoEnrichedBucketsError& e) {  // tools/projmotif.cpp:213-228
        std::cerr << "error: " << e.what() << '\n';
        return 3;
    } catch (const pmx::ParseError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 4;
    } catch (const pmx::IoError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 4;
    } catch (const pmx::ParamError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    }
}
