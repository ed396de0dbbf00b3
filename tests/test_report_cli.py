"""the `find`/`gen` command line, FASTA I/O and the schema-v1 JSON/TSV
report.  Formatting and parsing are compared byte for byte with fixtures produced by the
reference's own report.hpp / fasta.hpp (tests/golden/make_report_golden.cpp); the end-to-end CLI
run (GPU) must equal the reference's report except for wall_ms and the FP32-tolerance field."""
import json
import os
import re
import subprocess

import pytest

from conftest import EXPECTATION_TOL, REPO


@pytest.fixture(scope="module")
def report_golden():
    with open(os.path.join(REPO, "tests", "golden", "report_golden.json")) as f:
        return json.load(f)


def _compile(pm, source, exe):
    subprocess.run(["g++", "-std=c++17", "-O0", "-I" + os.path.join(REPO, "include"), os.path.join(REPO, source),
                    "-L" + pm.PKG_DIR, "-lpm_b200", "-Wl,-rpath," + pm.PKG_DIR, "-o", exe], check=True)
    return exe


@pytest.fixture(scope="module")
def report_test(pm):
    return _compile(pm, "tests/cpp/report_test.cpp", "/tmp/pm_report_test")


@pytest.fixture(scope="module")
def cli(pm):
    return _compile(pm, "tools/projmotif_b200.cpp", "/tmp/projmotif_b200_cli")


def test_report_rendering_is_byte_identical(report_test, report_golden, tmp_path):
    for i, case in enumerate(report_golden["results"]):
        f = case["fields"]
        path = tmp_path / f"fields{i}.txt"
        lines = [f"{k}={','.join(map(str, v)) if isinstance(v, list) else repr(v) if isinstance(v, float) else v}"
                 for k, v in f.items()]
        path.write_text("\n".join(lines) + "\n")
        out = subprocess.run([report_test, "render", str(path)], capture_output=True, text=True, check=True).stdout
        got_json, got_tsv = out.split("\x1e")
        assert got_json == case["json"]
        assert got_tsv == case["tsv"]


def test_fasta_parser_matches_reference(report_test, report_golden, tmp_path):
    for i, case in enumerate(report_golden["fasta"]):
        path = tmp_path / f"in{i}.fa"
        path.write_bytes(case["text"].encode())
        out = subprocess.run([report_test, "fasta", str(path)], capture_output=True, text=True, check=True).stdout
        if "error" in case:
            assert out.strip() == case["error"], case["text"]
        else:
            lines = out.split("\n")
            assert lines[0] == "ok"
            got = [tuple(x.split("\t")) for x in lines[1:] if x != ""]
            assert got == list(zip(case["names"], case["seqs"])), case["text"]


def test_gen_matches_reference(report_test, cli, report_golden, tmp_path):
    g = report_golden["gen"]
    out = subprocess.run([report_test, "gen"] + [str(g[k]) for k in ("t", "n", "l", "d", "seed")],
                         capture_output=True, text=True, check=True).stdout
    fasta, truth = out.split("\x1e")
    assert fasta == g["fasta"] and truth == g["truth"]
    target = tmp_path / "g.fasta"
    r = subprocess.run([cli, "gen", "--t", str(g["t"]), "--n", str(g["n"]), "--l", str(g["l"]), "--d", str(g["d"]),
                        "--seed", str(g["seed"]), "-o", str(target)], capture_output=True, text=True)
    assert r.returncode == 0 and "wrote" in r.stderr
    assert target.read_text() == g["fasta"]
    assert (tmp_path / "g.fasta.truth.json").read_text() == g["truth"]


def test_cli_usage_and_io_errors(cli, tmp_path):
    # exit codes of tools/projmotif.cpp:213-228: 2 usage/parameter, 4 parse/I-O
    assert subprocess.run([cli]).returncode == 2
    assert subprocess.run([cli, "find", "--l", "8", "--d", "1"], capture_output=True).returncode == 2
    assert subprocess.run([cli, "find", "-i", "/nonexistent.fa", "--l", "8", "--d", "1"], capture_output=True).returncode == 4
    bad = tmp_path / "bad.fa"
    bad.write_text("ACGT\n")
    assert subprocess.run([cli, "find", "-i", str(bad), "--l", "3", "--d", "1"], capture_output=True).returncode == 4
    assert subprocess.run([cli, "find", "-i", str(bad), "--l", "x", "--d", "1"], capture_output=True).returncode == 2
    assert subprocess.run([cli, "oracle"], capture_output=True).returncode == 2


@pytest.mark.gpu
def test_cli_find_matches_reference_report(cli, report_test, report_golden, tmp_path):
    c = report_golden["find_case"]
    fasta = tmp_path / "in.fa"
    out = subprocess.run([report_test, "gen", str(c["t"]), str(c["n"]), str(c["l"]), str(c["d"]), str(c["inst_seed"])],
                         capture_output=True, text=True, check=True).stdout
    fasta.write_text(out.split("\x1e")[0])
    args = [cli, "find", "-i", str(fasta), "--l", str(c["l"]), "--d", str(c["d"]), "--k", str(c["k"]), "--s", str(c["s"]),
            "--m", str(c["m"]), "--seed", str(c["seed"]), "--no-early-stop"]
    r = subprocess.run(args, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    want = report_golden["results"][0]["json"]
    got_doc, want_doc = json.loads(r.stdout), json.loads(want)
    assert abs(got_doc["best"]["expectation"] - want_doc["best"]["expectation"]) <= EXPECTATION_TOL

    def neutral(text):  # blank out the two fields that legitimately differ
        text = re.sub(r'"wall_ms": [^\n]+', '"wall_ms": 0', text)
        return re.sub(r'"expectation": [^\n]+', '"expectation": 0,', text)
    assert neutral(r.stdout) == neutral(want)
    tsv = subprocess.run(args + ["--format", "tsv"], capture_output=True, text=True)
    assert tsv.returncode == 0
    head, row = tsv.stdout.strip().split("\n")
    want_head, want_row = report_golden["results"][0]["tsv"].strip().split("\n")
    assert head == want_head
    g, w = row.split("\t"), want_row.split("\t")
    assert g[:2] == w[:2] and g[3:8] == w[3:8] and abs(float(g[2]) - float(w[2])) <= EXPECTATION_TOL
    # exit code 3 when nothing is ever enriched (tools/projmotif.cpp:213-215)
    none = subprocess.run([cli, "find", "-i", str(fasta), "--l", "8", "--d", "1", "--s", "500", "--m", "2"], capture_output=True)
    assert none.returncode == 3
    # stdin input
    piped = subprocess.run(args[:3] + ["-"] + args[4:], input=fasta.read_text(), capture_output=True, text=True)
    assert piped.returncode == 0 and neutral(piped.stdout) == neutral(want)
