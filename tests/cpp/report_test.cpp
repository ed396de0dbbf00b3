// Host-only driver for the report / FASTA parity tests (tests/test_report_cli.py):
//   report_test render <fields-file>   -> render_result_json, "\x1e", render_result_tsv
//   report_test fasta <text-file>      -> "ok" + name/sequence lines, or the error type name
//   report_test gen t n l d seed       -> serialize_fasta, "\x1e", truth_json
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>

#include "projmotif_b200.hpp"

using namespace projmotif_b200;

static std::string slurp(const char* path) {
    std::ifstream in(path, std::ios::binary);
    std::ostringstream b;
    b << in.rdbuf();
    return b.str();
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "";
    if (mode == "render" && argc > 2) {
        std::map<std::string, std::string> f;
        std::istringstream in(slurp(argv[2]));
        std::string line;
        while (std::getline(in, line)) {
            const std::size_t eq = line.find('=');
            if (eq != std::string::npos) f[line.substr(0, eq)] = line.substr(eq + 1);
        }
        RunResult r;
        r.params.l = std::stoi(f["l"]);
        r.params.d = std::stoi(f["d"]);
        r.params.k = std::stoi(f["k"]);
        r.params.s = std::stoi(f["s"]);
        r.params.m = std::stoll(f["m"]);
        r.params.q = std::stod(f["q"]);
        r.seed = std::stoull(f["seed"]);
        r.best.consensus = f["motif"];
        r.best.score = std::stoi(f["score"]);
        r.best.expectation = std::stod(f["expectation"]);
        std::istringstream ps(f["positions"]);
        std::string tok;
        while (std::getline(ps, tok, ',')) {
            if (!tok.empty()) r.best.positions.push_back(std::stoi(tok));
        }
        r.best.source_bucket = std::stoull(f["source_bucket"]);
        r.best_trial = std::stoll(f["trial"]);
        r.trials_run = std::stoll(f["trials_run"]);
        r.buckets_enriched = std::stoll(f["buckets_enriched"]);
        r.wall_ms = std::stod(f["wall_ms"]);
        std::cout << render_result_json(r) << '\x1e' << render_result_tsv(r);
        return 0;
    }
    if (mode == "fasta" && argc > 2) {
        try {
            const SequenceSet s = parse_fasta(slurp(argv[2]));
            std::cout << "ok\n";
            for (int i = 1; i <= s.count(); ++i) std::cout << s.name(i) << '\t' << s.sequence(i) << '\n';
        } catch (const RecordWithoutSequenceError&) {
            std::cout << "RecordWithoutSequenceError\n";
        } catch (const FastaFormatError&) {
            std::cout << "FastaFormatError\n";
        } catch (const EmptyInputError&) {
            std::cout << "EmptyInputError\n";
        } catch (const UnknownSymbolError&) {
            std::cout << "UnknownSymbolError\n";
        }
        return 0;
    }
    if (mode == "gen" && argc > 6) {
        const PlantedInstance inst = generate_planted(std::stoi(argv[2]), std::stoi(argv[3]), std::stoi(argv[4]),
                                                      std::stoi(argv[5]), std::stoull(argv[6]));
        std::cout << serialize_fasta(inst.sequences) << '\x1e' << truth_json(inst);
        return 0;
    }
    return 64;
}
