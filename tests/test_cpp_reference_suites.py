"""The reference's own Catch2 suites, compiled UNMODIFIED against the source-compatibility headers
(include/chunktrain/*.hpp -> the C++ facade include/oomb.hpp -> liboomb.so) and run on the B200.

    /root/reference/proj/tests/test_attention.cpp   (score / select / forward / backward, 12 cases)
    /root/reference/proj/tests/test_paged_kv.cpp    (page manager, 17 cases)

They are compiled by __graft_entry__.build() in the build container, where /root/reference exists,
with a minimal Catch2 stand-in (tests/cpp/shim; Catch2 is not installed here); the binaries and a
manifest of the SHA-256 of the sources they were built from travel to the GPU box in-tree.

PagedCache<double> runs an OOMB_F64 pool (double pages and arithmetic on the device), so the
reference's f64 cases (e.g. the all-pages backward at 1e-10 against its naive oracle) hold too:
every case must pass.
"""
import hashlib
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2602_02108_b200")
OUT = os.path.join(PKG, "_build")
REF_TESTS = "/root/reference/proj/tests"
SUITES = ("test_attention", "test_paged_kv")
MANIFEST = os.path.join(OUT, "reference_suites.json")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build_reference_suites() -> dict:
    """Compile the reference suites (only where /root/reference is present)."""
    if not os.path.isdir(REF_TESTS):
        return {}
    from oracle.oracle import build_port
    from paper_2602_02108_b200.build import build
    build()
    build_port()
    os.makedirs(OUT, exist_ok=True)
    manifest = {}
    for name in SUITES:
        src = os.path.join(REF_TESTS, name + ".cpp")
        binary = os.path.join(OUT, "ref_" + name)
        cmd = ["g++", "-std=c++20", "-O1", "-Wall", f"-I{ROOT}/tests/cpp/shim", f"-I{ROOT}/include",
               f"-I{CUDA}/include", src, os.path.join(ROOT, "tests", "cpp", "reference_suites_main.cpp"), "-o",
               binary, f"-L{PKG}", "-loomb", f"-L{ROOT}/oracle", "-loomb_oracle", f"-L{CUDA}/lib64", "-lcudart",
               f"-Wl,-rpath,{PKG}:{ROOT}/oracle:{CUDA}/lib64"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"reference suite {name} does not compile against include/chunktrain:\n{r.stderr}")
        manifest[name] = {"source": src, "sha256": hashlib.sha256(open(src, "rb").read()).hexdigest(),
                          "binary": os.path.relpath(binary, ROOT)}
    with open(MANIFEST, "w") as f:
        json.dump(manifest, f, indent=1)
    return manifest


def _run(name, filt=None):
    binary = os.path.join(OUT, "ref_" + name)
    if not os.path.exists(binary):
        pytest.skip("reference suites not built (build() runs where /root/reference exists)")
    r = subprocess.run([binary] + ([filt] if filt else []), capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    results = {}
    for line in r.stdout.splitlines():
        if line.startswith("PASS  ") or line.startswith("FAIL  "):
            results[line[6:]] = line[:4]
    return r, results


def test_reference_suites_manifest():
    """The binaries were built from the reference's sources, unmodified (hash recorded at build)."""
    if not os.path.exists(MANIFEST):
        pytest.skip("reference suites not built")
    m = json.load(open(MANIFEST))
    assert set(m) == set(SUITES)
    if os.path.isdir(REF_TESTS):
        for name, e in m.items():
            assert hashlib.sha256(open(e["source"], "rb").read()).hexdigest() == e["sha256"], name


def test_reference_contiguous_cases_cpu():
    """Host-only cases of test_paged_kv.cpp (the contiguous-growth baseline) run without a GPU."""
    r, res = _run("test_paged_kv", "contiguous")
    assert r.returncode == 0 and len(res) == 2 and all(v == "PASS" for v in res.values()), r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", SUITES)
def test_reference_suite_on_b200(name):
    r, res = _run(name)
    assert res, r.stdout + r.stderr
    failed = {k for k, v in res.items() if v == "FAIL"}
    assert not failed, f"failed: {failed}"
    assert len(res) >= (12 if name == "test_attention" else 17)
