"""The reference's OWN test suites run through the B200 framework's C++ API
(VERDICT r1 item 7).

`make` compiles /root/reference/proj/tests/{test_dataset,test_eval,
test_graph_build,test_kd_forest,test_search}.cpp and acceptance.cpp unchanged
against include/annkit_b200.hpp (tests/cpp/shim maps "annkit/*.hpp" to it;
tests/cpp/doctest/doctest.h is our doctest-compatible harness, since the
reference does not ship doctest) into tests/cpp/_refsuite/, linked to
libannkit_facade.so -> libannkit_b200.so.  The same unit sources are also built
against the reference library itself (oracle/_ref/unit_ref), which pins the
harness: every reference test case passes there.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "tests", "cpp", "_refsuite")
REF_UNIT = os.path.join(ROOT, "oracle", "_ref", "unit_ref")


def _cases(out):
    return {m.group(2): m.group(1) for m in re.finditer(r"^\[case\] (PASS|FAIL|SKIP) (.+)$", out, re.M)}


@pytest.mark.skipif(not os.path.exists(REF_UNIT), reason="oracle/_ref/unit_ref not built (no /root/reference)")
def test_harness_runs_reference_suite_on_reference_library():
    p = subprocess.run([REF_UNIT], capture_output=True, text=True, timeout=600)
    cases = _cases(p.stdout)
    assert len(cases) == 52 and all(v == "PASS" for v in cases.values()), p.stdout[-2000:] + p.stderr[-2000:]
    assert p.returncode == 0


@pytest.mark.gpu
def test_reference_unit_suite_through_b200_api():
    exe = os.path.join(SUITE, "unit")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/_refsuite not built (needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=1200, cwd=ROOT)
    cases = _cases(p.stdout)
    failed = sorted(k for k, v in cases.items() if v != "PASS")
    assert len(cases) == 52, p.stdout[-3000:]
    assert not failed, f"{failed}\n{p.stderr[-4000:]}"
    assert p.returncode == 0


@pytest.mark.gpu
def test_reference_acceptance_runner_through_b200_api():
    exe = os.path.join(SUITE, "acceptance")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/_refsuite not built (needs /root/reference at build time)")
    cli = os.path.join(ROOT, "paper_1609_07228_b200", "annkit")
    p = subprocess.run([exe, "--cli", cli], capture_output=True, text=True, timeout=1800, cwd=ROOT)
    out = p.stdout
    res = {int(m.group(2)): m.group(1) for m in re.finditer(r"^(PASS|FAIL) criterion (\d+):", out, re.M)}
    assert sorted(res) == list(range(1, 10)), out
    # criterion 2 (10% of n(n-1)/2 comparisons to 0.90 on 10k x 128 uniform data) fails
    # by design, in the reference too (proj/README.md:119-127, proj/test_output.txt:11)
    assert res[2] == "FAIL"
    assert all(res[c] == "PASS" for c in res if c != 2), out
    # the reference's recorded known answers (proj/test_output.txt:9-20), bit-exact
    for golden in ("29454671 dist comps = 58.9%", "efanna 29454671 < random-descent 37263414 < nn-expansion never "
                   "(plateau 0.7000)", "recall 0.9440 at 1285 comps/query",
                   "[P=50: 0.851 >= 0.787] [P=100: 0.944 >= 0.898] [P=200: 0.970 >= 0.947] [P=300: 0.978 >= 0.968]"
                   " [P=400: 0.990 >= 0.976] [P=600: 0.996 >= 0.986]",
                   "graph acc 0.6090; accuracy_vs_k 10->0.6090 100->1.0000 (delta 0.3910, need >= 0.20); "
                   "recall drop 0.0370", "20/20 exact graphs", "crosses 0.90 at 4976057 comps = 10.0%",
                   "38 logged steps across 6 runs, 0 violations", "6 command pairs byte-identical"):
        assert golden in out, golden
