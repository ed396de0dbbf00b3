// Generates tests/golden/report_golden.json from the UNMODIFIED reference report.hpp / fasta.hpp /
// planted.hpp (build container only; needs an nlohmann json.hpp on the include path):
//   g++ -std=c++20 -O1 -I/root/reference/proj/include -I<dir with json.hpp> tests/golden/make_report_golden.cpp -o /tmp/mrg && /tmp/mrg > tests/golden/report_golden.json
// The only json.hpp in this image is cudnn-frontend's copy of nlohmann 3.11.3 with one local patch ("Custom from FE":
// integer arrays printed inline); the fixture was generated against a temp copy with the stock condition
// `if (pretty_print)` restored at that site, i.e. upstream 3.11.3 behaviour.
#include <iostream>
#include <json.hpp>
#include <projmotif/driver.hpp>
#include <projmotif/fasta.hpp>
#include <projmotif/planted.hpp>
#include <projmotif/report.hpp>

using namespace projmotif;
using nlohmann::ordered_json;

static ordered_json result_case(RunResult r, double wall_ms) {
    r.wall_ms = wall_ms;
    ordered_json c;
    c["fields"] = {{"l", r.params.l}, {"d", r.params.d}, {"k", r.params.k}, {"s", r.params.s}, {"m", r.params.m},
                   {"q", r.params.q}, {"seed", r.seed}, {"motif", r.best.consensus}, {"score", r.best.score},
                   {"expectation", r.best.expectation}, {"positions", r.best.positions},
                   {"source_bucket", r.best.source_bucket}, {"trial", r.best_trial}, {"trials_run", r.trials_run},
                   {"buckets_enriched", r.buckets_enriched}, {"wall_ms", r.wall_ms}};
    c["json"] = render_result_json(r);
    c["tsv"] = render_result_tsv(r);
    return c;
}

static ordered_json parse_case(const std::string& text) {
    ordered_json c;
    c["text"] = text;
    try {
        const SequenceSet s = parse_fasta(std::string_view(text));
        std::vector<std::string> names, seqs;
        for (int i = 1; i <= s.count(); ++i) {
            names.push_back(s.name(i));
            seqs.push_back(s.sequence(i));
        }
        c["names"] = names;
        c["seqs"] = seqs;
    } catch (const RecordWithoutSequenceError&) {
        c["error"] = "RecordWithoutSequenceError";
    } catch (const FastaFormatError&) {
        c["error"] = "FastaFormatError";
    } catch (const EmptyInputError&) {
        c["error"] = "EmptyInputError";
    } catch (const UnknownSymbolError&) {
        c["error"] = "UnknownSymbolError";
    }
    return c;
}

int main() {
    ordered_json doc;
    {
        const PlantedInstance inst = generate_planted(12, 120, 8, 1, 5);
        RunConfig cfg;
        cfg.l = 8; cfg.d = 1; cfg.k = 5; cfg.s = 3; cfg.m = 6; cfg.seed = 3; cfg.early_stop = false;
        const RunResult r = run(cfg, inst.sequences);
        doc["results"].push_back(result_case(r, 28.146));
        RunResult r2 = r;
        r2.best.expectation = 8.0;  // integral double
        r2.params.q = 0.5;
        r2.best.positions = {1};
        r2.seed = 18446744073709551615ULL;
        doc["results"].push_back(result_case(r2, 0.001));
        RunResult r3 = r;
        r3.best.expectation = 1.0 / 3.0;
        r3.best.positions = {};
        doc["results"].push_back(result_case(r3, 123456.789));
        doc["find_case"] = {{"t", 12}, {"n", 120}, {"l", 8}, {"d", 1}, {"inst_seed", 5}, {"k", 5}, {"s", 3}, {"m", 6}, {"seed", 3}};
    }
    {
        const PlantedInstance inst = generate_planted(3, 70, 8, 1, 5);
        doc["gen"] = {{"t", 3}, {"n", 70}, {"l", 8}, {"d", 1}, {"seed", 5}, {"fasta", serialize_fasta(inst.sequences)}, {"truth", truth_json(inst)}};
    }
    for (const char* text : {">a\nACGT\nAC\n>b desc here\nttga\n", ">  spaced\r\nAC GT\r\n\r\n>x\r\nA\tC\r\n", "ACGT\n", ">only\n", ">a\nACGT\n>b\n",
                             "", "\n\n", ">a\nACNT\n", ">a\nACGT", ">\nAC\n"}) {
        doc["fasta"].push_back(parse_case(text));
    }
    std::cout << doc.dump(1) << "\n";
}
