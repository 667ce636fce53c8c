"""The C++ drop-in API (include/epi3/api.hpp -> libepi3.so -> libepi3cu.so)
and the CLI built on it, exercised the way the reference's C++ tests and
cli_test.cpp exercise the reference."""
import json
import subprocess
import tempfile
from pathlib import Path

import pytest

from helpers import product_dataset, ref_hits
from paper_2201_10956_b200 import build, epi3

ROOT = Path(__file__).resolve().parents[1]


def _compile_api_test(tmp: Path) -> Path:
    exe = tmp / "api_test"
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "cpp" / "api_test.cpp"), "-o", str(exe),
                    f"-L{build.PKG}", "-lepi3", "-lepi3cu", f"-Wl,-rpath,{build.PKG}"],
                   check=True)
    return exe


def test_api_test_compiles_against_the_dropin_headers():
    with tempfile.TemporaryDirectory() as d:
        assert _compile_api_test(Path(d)).exists()


def test_cli_usage_and_domain_exit_codes():
    # cli_test.cpp:62-72, 120-132: usage/domain errors exit 2
    r = subprocess.run([str(build.CLI)], capture_output=True)
    assert r.returncode == 2
    r = subprocess.run([str(build.CLI), "generate", "--snps", "10", "--samples", "10",
                        "--maf", "0.9", "--out", "/tmp/never.epi3"], capture_output=True)
    assert r.returncode == 2


@pytest.mark.gpu
def test_cpp_api_suite(golden_cases):
    case = golden_cases["cfg1"]
    with tempfile.TemporaryDirectory() as d:
        exe = _compile_api_test(Path(d))
        f = Path(d) / "cfg1.epi3"
        epi3.write_packed(f, product_dataset(case))
        best = case["search"]["best"]["triple"]
        r = subprocess.run([str(exe), str(f), *map(str, best)], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cli_detect_matches_reference(golden_cases):
    case = golden_cases["cfg1"]
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "cfg1.epi3"
        epi3.write_packed(f, product_dataset(case))
        r = subprocess.run([str(build.CLI), "detect", "--in", str(f), "--json"],
                           capture_output=True, text=True, check=True)
        got = json.loads(r.stdout)
        expect = ref_hits(case["search"])
        assert [tuple(h["triple"]) for h in got["top"]] == [t for _, t in expect]
        assert [h["score"] for h in got["top"]] == [s for s, _ in expect]
        txt = subprocess.run([str(build.CLI), "detect", "--in", str(f)], capture_output=True,
                             text=True, check=True).stdout
        b = case["search"]["best"]
        assert f"best ({b['triple'][0]},{b['triple'][1]},{b['triple'][2]}) k2={b['score']:.9f}" in txt


@pytest.mark.gpu
def test_cli_detect_text_input_binarizes_on_device():
    """A text genotype file goes through run_search(GenotypeMatrix) (binarize on
    the GPU) and reports exactly what the packed file of the same data does."""
    with tempfile.TemporaryDirectory() as d:
        t, p = Path(d) / "g.txt", Path(d) / "g.epi3"
        for out, fmt in ((t, "text"), (p, "packed")):
            subprocess.run([str(build.CLI), "generate", "--snps", "40", "--samples", "900",
                            "--seed", "9", "--plant", "4,17,31:1,1,1:0.9,0.1", "--format", fmt, "--out", str(out)],
                           check=True, capture_output=True)
        rt = json.loads(subprocess.run([str(build.CLI), "detect", "--in", str(t), "--json"],
                                       capture_output=True, text=True, check=True).stdout)
        rp = json.loads(subprocess.run([str(build.CLI), "detect", "--in", str(p), "--json"],
                                       capture_output=True, text=True, check=True).stdout)
        for k in ("snps", "samples", "controls", "cases", "best", "top"):
            assert rt[k] == rp[k], k


# ---------------------------------------------------------------------------
# The reference CLI's own test suite (proj/tests/cli_test.cpp:46-224), ported
# assertion for assertion: the same command lines against epi3_cli.
# ---------------------------------------------------------------------------


def _cli(args: str):
    r = subprocess.run(f"{build.CLI} {args} 2>&1", shell=True, capture_output=True, text=True)
    return r.returncode, r.stdout


def test_cli_generate_is_deterministic(tmp_path):
    # cli_test.cpp:46-56
    a, b = tmp_path / "gen_a.txt", tmp_path / "gen_b.txt"
    flags = "generate --snps 10 --samples 100 --maf 0.3 --seed 1 --out "
    assert _cli(flags + str(a))[0] == 0
    assert _cli(flags + str(b))[0] == 0
    text = a.read_text()
    assert text.split("\n")[0] == "#SNPS=10 SAMPLES=100"
    assert a.read_bytes() == b.read_bytes()


def test_cli_generate_rejects_bad_parameters(tmp_path):
    # cli_test.cpp:58-68
    out = tmp_path / "gen_bad.txt"
    assert _cli(f"generate --snps 10 --samples 100 --maf 0.9 --out {out}")[0] == 2
    assert _cli(f"generate --snps 10 --samples 100 --plant 1,1,2:0,0,0:0.9,0.1 --out {out}")[0] == 2
    assert _cli(f"generate --samples 100 --out {out}")[0] == 2  # missing required --snps
    assert _cli(f"generate --snps 10 --samples 100 --bogus 1 --out {out}")[0] == 2
    assert _cli(f"generate --snps 10 --samples 100 --format xml --out {out}")[0] == 2


def test_cli_generate_plant_line(tmp_path):
    # epi3_main.cpp:96-101: the plant spec is parsed in full and echoed
    out = tmp_path / "p.txt"
    rc, txt = _cli(f"generate --snps 24 --samples 64 --maf 0.5 --seed 3 "
                   f"--plant 4,11,19:1,1,1:0.9,0.1 --out {out}")
    assert rc == 0
    assert f"wrote {out}: snps=24 samples=64 format=text" in txt
    assert "planted triple (4,11,19) target (1,1,1) p=0.9/0.1" in txt


@pytest.mark.gpu
def test_cli_detect_planted_and_block_parameters(tmp_path):
    # cli_test.cpp:74-103
    data = tmp_path / "detect.txt"
    assert _cli(f"generate --snps 24 --samples 1024 --maf 0.5 --seed 3 "
                f"--plant 4,11,19:1,1,1:0.9,0.1 --out {data}")[0] == 0
    rc, v4 = _cli(f"detect --in {data} --variant v4 --threads 2")
    assert rc == 0
    assert "best (4,11,19)" in v4
    assert "block=<5,400>" in v4
    assert "variant=v4 threads=2 block=<5,400> sched=256 lanes=8" in v4
    rc, v1 = _cli(f"detect --in {data} --variant v1 --threads 2")
    assert rc == 0

    def best_line(s):
        at = s.index("best (")
        return s[at:s.index("\n", at)]
    assert best_line(v1) == best_line(v4)
    line = best_line(v4)
    dot = line.index(".", line.index("k2="))
    assert len(line) - dot - 1 == 9


@pytest.mark.gpu
def test_cli_detect_json_document(tmp_path):
    # cli_test.cpp:105-118
    data = tmp_path / "detect_json.txt"
    assert _cli(f"generate --snps 12 --samples 200 --seed 5 --out {data}")[0] == 0
    rc, out = _cli(f"detect --in {data} --threads 1 --top-k 3 --json")
    assert rc == 0
    j = json.loads(out)
    assert j["snps"] == 12 and j["samples"] == 200
    assert "triple" in j["best"]
    assert len(j["top"]) == 3
    assert j["block"]["snps"] == 5 and j["block"]["samples"] == 400
    assert j["variant"] == "v4" and j["threads"] == 1
    assert j["stats"]["combinations"] == epi3.num_combinations(12, 3)
    assert sum(j["stats"]["per_thread_work"]) == epi3.num_combinations(12, 3)


@pytest.mark.gpu
def test_cli_detect_exit_codes(tmp_path):
    # cli_test.cpp:120-132
    data = tmp_path / "detect_codes.txt"
    assert _cli(f"generate --snps 8 --samples 64 --seed 2 --out {data}")[0] == 0
    assert _cli("detect --in /nonexistent/path.txt")[0] == 1
    assert _cli(f"detect --in {data} --l1-kb 1 --l1-ways 8 --ft-ways 1 --block-ways 1")[0] == 2
    assert _cli(f"detect --in {data} --variant v9")[0] == 2


@pytest.mark.gpu
def test_cli_packed_detects_like_text(tmp_path):
    # cli_test.cpp:134-150
    text, packed = tmp_path / "fmt.txt", tmp_path / "fmt.bin"
    assert _cli(f"generate --snps 16 --samples 333 --seed 11 --maf 0.4 --out {text}")[0] == 0
    assert _cli(f"generate --snps 16 --samples 333 --seed 11 --maf 0.4 --format packed "
                f"--out {packed}")[0] == 0
    ra, a = _cli(f"detect --in {text} --threads 1")
    rb, b = _cli(f"detect --in {packed} --threads 1")
    assert ra == 0 and rb == 0
    assert a[a.index("best"):a.index("stats:")] == b[b.index("best"):b.index("stats:")]


@pytest.mark.gpu
def test_cli_verify_clean_and_corrupted(tmp_path):
    # cli_test.cpp:152-198
    data = tmp_path / "verify.bin"
    assert _cli(f"generate --snps 20 --samples 150 --seed 17 --format packed --out {data}")[0] == 0
    rc, ok = _cli(f"verify --in {data}")
    assert rc == 0, ok
    assert "FAIL" not in ok
    assert "tables v1 vs oracle" in ok and "search tpc vs oracle" in ok
    assert ok.count("PASS") == 10
    b = bytearray(data.read_bytes())
    n0 = int.from_bytes(b[16:24], "little")
    w0 = (n0 + 63) // 64
    injected = False
    for k in range(8 * w0):
        if b[32 + 8 * w0 + k]:
            b[32 + k] |= b[32 + 8 * w0 + k]
            injected = True
            break
    assert injected
    data.write_bytes(bytes(b))
    rc, bad = _cli(f"verify --in {data}")
    assert rc == 1 and "FAIL" in bad
    data.write_bytes(bytes(b[:-3]))
    assert _cli(f"verify --in {data}")[0] == 1
    big = tmp_path / "verify_big.txt"
    assert _cli(f"generate --snps 70 --samples 40 --seed 1 --out {big}")[0] == 0
    assert _cli(f"verify --in {big}")[0] == 1
    assert _cli(f"verify --in {big} --max-snps 70")[0] == 0


@pytest.mark.gpu
def test_cli_bench_reports(tmp_path):
    # cli_test.cpp:200-224 (+ bench.cpp:72-107 columns)
    data = tmp_path / "bench.txt"
    assert _cli(f"generate --snps 14 --samples 256 --seed 23 --out {data}")[0] == 0
    rc, csv = _cli(f"bench --in {data} --variant v2 --repeats 2 --threads 1")
    assert rc == 0
    assert csv.count("\n") == 2
    assert csv.startswith("variant,M,N,threads,elapsed_s,elements,eps,eps_per_thread,"
                          "model_ops,model_bytes,ai\n")
    row = csv.split("\n")[1].split(",")
    assert row[0] == "v2" and row[1] == "14" and row[2] == "256" and row[3] == "1"
    assert int(row[5]) == epi3.num_combinations(14, 3) * 256
    assert row[8] == "57"
    rc, js = _cli(f"bench --in {data} --variant v4 --repeats 2 --threads 1 --format json")
    assert rc == 0
    j = json.loads(js)
    assert j["variant"] == "v4" and len(j["repeats_s"]) == 2
    out = tmp_path / "bench_out.csv"
    assert _cli(f"bench --in {data} --repeats 1 --threads 1 --out {out}")[0] == 0
    assert out.read_text().startswith("variant,")
