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
def test_cli_verify_and_bench():
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "g.epi3"
        subprocess.run([str(build.CLI), "generate", "--snps", "24", "--samples", "700",
                        "--seed", "4", "--plant", "3,11,19", "--out", str(f)], check=True)
        r = subprocess.run([str(build.CLI), "verify", "--in", str(f)], capture_output=True,
                           text=True)
        assert r.returncode == 0 and r.stdout.count("PASS") == 2, r.stdout
        r = subprocess.run([str(build.CLI), "bench", "--in", str(f), "--repeats", "2",
                            "--format", "json"], capture_output=True, text=True, check=True)
        rep = json.loads(r.stdout)
        assert rep["elements"] == epi3.num_combinations(24, 3) * 700 and rep["eps"] > 0


@pytest.mark.gpu
def test_cli_detect_text_input_binarizes_on_device():
    """A text genotype file goes through run_search(GenotypeMatrix) (binarize on
    the GPU) and reports exactly what the packed file of the same data does."""
    with tempfile.TemporaryDirectory() as d:
        t, p = Path(d) / "g.txt", Path(d) / "g.epi3"
        for out, fmt in ((t, "text"), (p, "packed")):
            subprocess.run([str(build.CLI), "generate", "--snps", "40", "--samples", "900",
                            "--seed", "9", "--plant", "4,17,31", "--format", fmt, "--out", str(out)],
                           check=True, capture_output=True)
        rt = json.loads(subprocess.run([str(build.CLI), "detect", "--in", str(t), "--json"],
                                       capture_output=True, text=True, check=True).stdout)
        rp = json.loads(subprocess.run([str(build.CLI), "detect", "--in", str(p), "--json"],
                                       capture_output=True, text=True, check=True).stdout)
        for k in ("snps", "samples", "controls", "cases", "best", "top"):
            assert rt[k] == rp[k], k
