"""the exact solvers of oracle.hpp (median_string on the device, naive_mfp on the
host), the `oracle` / `bench` command lines and the benchmark() TSV harness (driver.hpp:253-302), against
fixtures produced by the reference itself (tests/golden/make_bench_golden.cpp) and against the CPU oracle."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import REPO
from oracle import pmo


@pytest.fixture(scope="module")
def bench_golden():
    with open(os.path.join(REPO, "tests", "golden", "bench_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def cli(pm):
    exe = "/tmp/projmotif_b200_cli2"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I" + os.path.join(REPO, "include"), os.path.join(REPO, "tools/projmotif_b200.cpp"),
                    "-L" + pm.PKG_DIR, "-lpm_b200", "-Wl,-rpath," + pm.PKG_DIR, "-o", exe], check=True)
    return exe


def test_oracle_port_matches_reference_fixtures(port, bench_golden):
    """CPU: the plain-C restatement of the exact solvers reproduces the reference's answers."""
    for g in bench_golden["oracle"][:3]:
        ss, _, _ = port.generate_planted(g["t"], g["n"], g["l"], g["d"], g["seed"])
        assert port.median_string(ss, g["l"]) == (g["median"], g["total_distance"])
        if "naive_score" in g:
            assert port.naive_mfp(ss, g["l"]) == (g["naive_positions"], g["naive_score"], g["naive_consensus"])
    ss = pmo.SeqSet.from_strings(["ACGTAC", "GGTACA"])
    with pytest.raises(pmo.OracleError) as e:
        port.median_string(ss, 5, limit=100)
    assert e.value.code == 11  # SearchSpaceTooLargeError
    with pytest.raises(pmo.OracleError) as e:
        port.naive_mfp(ss, 3, limit=5)
    assert e.value.code == 11


@pytest.mark.gpu
def test_median_string_matches_reference_and_oracle(pm, ctx, best_oracle, bench_golden):
    for g in bench_golden["oracle"]:
        ss, _, _ = best_oracle.generate_planted(g["t"], g["n"], g["l"], g["d"], g["seed"])
        ctx.set_sequences(ss.bases, ss.offs)
        assert ctx.median_string(g["l"]) == (g["median"], g["total_distance"])
        # the reported distance is the XOR/popcount scan of the reported median
        assert ctx.hamming_scan(g["median"], 0)[1] == g["total_distance"]
    rng = np.random.default_rng(8)
    for _ in range(8):  # ragged random sets, ties between candidates resolved to the smallest code
        l = int(rng.integers(1, 8))
        ss = pmo.SeqSet.from_strings(["".join(rng.choice(list("ACGT"), int(rng.integers(l, l + 30)))) for _ in range(int(rng.integers(1, 7)))])
        ctx.set_sequences(ss.bases, ss.offs)
        assert ctx.median_string(l) == best_oracle.median_string(ss, l)
    for l, limit, kind in ((5, 100, "SearchSpaceTooLargeError"), (13, 16777216, "SearchSpaceTooLargeError"),
                           (0, 10, "InvalidParamsError"), (32, 2 ** 63, "InvalidParamsError"), (40, 10, "InvalidParamsError")):
        ss = pmo.SeqSet.from_strings(["ACGT" * 12, "TTGACA" * 8])
        ctx.set_sequences(ss.bases, ss.offs)
        with pytest.raises(pm.PmError) as e:
            ctx.median_string(l, limit)
        assert e.value.kind == kind, (l, limit)


@pytest.mark.gpu
def test_median_string_validates_a_recovered_motif_at_scale(ctx, port):
    """(12,3) planted in 20 x 600: 4^12 candidates x 11,780 windows.  The exhaustive median cannot be farther
    from the sequences than the planted motif, and nothing run() reports can be closer than the median."""
    ss, motif, _ = port.generate_planted(20, 600, 12, 3, 42)
    ctx.set_sequences(ss.bases, ss.offs)
    median, dist = ctx.median_string(12)
    planted = ctx.hamming_scan(motif, 3)
    assert dist <= planted[1] and ctx.hamming_scan(median, 3)[1] == dist
    assert median == motif  # the planted motif is the exact median of this instance
    got = ctx.run(l=12, d=3, k=6, s=3, m=60, seed=7, early_stop=0)
    assert got["total_distance"] >= dist  # no candidate of the projection search can beat the exhaustive optimum
    assert (got["total_distance"] == dist) == (got["consensus"] == median) or got["total_distance"] == dist


@pytest.mark.gpu
def test_cli_oracle_and_bench_match_reference(cli, bench_golden, tmp_path):
    g = bench_golden["oracle"][0]
    fasta = tmp_path / "o.fa"
    r = subprocess.run([cli, "gen", "--t", str(g["t"]), "--n", str(g["n"]), "--l", str(g["l"]), "--d", str(g["d"]),
                        "--seed", str(g["seed"]), "-o", str(fasta)], capture_output=True, text=True)
    assert r.returncode == 0
    med = subprocess.run([cli, "oracle", "-i", str(fasta), "--l", str(g["l"]), "--method", "median"], capture_output=True, text=True)
    assert med.returncode == 0, med.stderr
    assert med.stdout == '{\n  "method": "median",\n  "median": "%s",\n  "total_distance": %d\n}\n' % (g["median"], g["total_distance"])
    nv = subprocess.run([cli, "oracle", "-i", str(fasta), "--l", str(g["l"])], capture_output=True, text=True)
    assert nv.returncode == 0, nv.stderr
    doc = json.loads(nv.stdout)
    assert list(doc) == ["method", "score", "positions", "consensus"]
    assert (doc["method"], doc["score"], doc["positions"], doc["consensus"]) == \
           ("naive", g["naive_score"], g["naive_positions"], g["naive_consensus"])
    assert subprocess.run([cli, "oracle", "-i", str(fasta), "--l", str(g["l"]), "--limit", "10"], capture_output=True).returncode == 2
    for b in bench_golden["bench"]:
        args = [cli, "bench", "--instances", str(b["instances"]), "--t", str(b["t"]), "--n", str(b["n"]), "--l", str(b["l"]),
                "--d", str(b["d"]), "--seed", str(b["seed"]), "--s", str(b["s"])] + (["--m", str(b["m"])] if b["m"] else [])
        r = subprocess.run(args, capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        rows = [line.split("\t") for line in r.stdout.strip().split("\n")]
        want = [line.split("\t") for line in b["tsv"].strip().split("\n")]
        assert rows[0] == want[0]
        assert [row[:6] for row in rows[1:]] == [row[:6] for row in want[1:]]
        assert all(float(v) >= 0 for row in rows[1:] for v in row[6:])
