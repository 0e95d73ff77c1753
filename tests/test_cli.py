"""The `annkit` command line (reference proj/tools/main.cpp).

Artifacts written by the B200 CLI — AKF1 forests, ground truth, graphs,
search results — must be byte-identical to what the reference library writes
for the same inputs (its own build_forest / brute_force / build_graph / search
followed by its own save_* writers, through oracle/_ref); CSV rows must carry
the same values except the timing columns.  The reference CLI binary itself
is not built: it needs the un-vendored CLI11 header (proj/CMakeLists.txt
`vendor/`), so parity is anchored on the library calls it makes.  The
reference's acceptance runner drives this CLI for its criterion 8
(tests/test_reference_suites.py).
"""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1609_07228_b200", "annkit")
needs_ref = pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")


def run(*args, ok=True):
    assert os.path.exists(CLI), "CLI not built (make)"
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)
    if ok:
        assert p.returncode == 0, p.stderr
    return p


def _bytes(p):
    with open(p, "rb") as fh:
        return fh.read()


def g10(x):
    """C++ `ostream << setprecision(10) << double` formatting."""
    return "%.10g" % x


def csv_rows(text):
    return [line.split(",") for line in text.splitlines() if line and not line.startswith("#")]


@pytest.fixture
def tmp():
    with tempfile.TemporaryDirectory() as d:
        yield d


# ------------------------------------------------------------------ CPU

def test_usage_errors():
    assert run("--help").returncode == 0
    assert run(ok=False).returncode == 2
    p = run("frobnicate", ok=False)
    assert p.returncode == 2 and "unknown subcommand" in p.stderr
    p = run("build-trees", "--base", "x.fvecs", ok=False)
    assert p.returncode == 2 and "is required" in p.stderr
    p = run("convert", "--out", "o.fvecs", ok=False)
    assert p.returncode == 2 and "exactly one of --in / --synthetic" in p.stderr
    p = run("convert", "--synthetic", "10x4", "--out", "o.fvecs", ok=False)
    assert p.returncode == 2 and "N:DIM:SEED" in p.stderr
    p = run("build-trees", "--base", "/nonexistent.fvecs", "--seed", 1, "--out", "f.akf", ok=False)
    assert p.returncode == 1 and "cannot open file" in p.stderr


@needs_ref
def test_convert_synthetic_and_copy_match_reference(tmp):
    r = O.load("reference")
    out = os.path.join(tmp, "syn.fvecs")
    p = run("convert", "--synthetic", "300:9:17", "--out", out)
    assert p.stdout == f"wrote 300x9 vectors to {out}\n"
    r.ref_save_fvecs(r.vs(r.gen_synthetic(300, 9, 17)), os.path.join(tmp, "ref.fvecs"))
    assert _bytes(out) == _bytes(os.path.join(tmp, "ref.fvecs"))
    # --limit keeps the first N records, for fvecs and ivecs
    run("convert", "--in", out, "--out", os.path.join(tmp, "cut.fvecs"), "--limit", 120)
    r.ref_save_fvecs(r.vs(r.gen_synthetic(300, 9, 17)[:120]), os.path.join(tmp, "refcut.fvecs"))
    assert _bytes(os.path.join(tmp, "cut.fvecs")) == _bytes(os.path.join(tmp, "refcut.fvecs"))
    ids = (np.arange(50 * 6, dtype=np.uint32) * 7919 % 1000).reshape(50, 6)
    r.ref_save_ivecs(ids, os.path.join(tmp, "a.ivecs"))
    p = run("convert", "--in", os.path.join(tmp, "a.ivecs"), "--out", os.path.join(tmp, "b.ivecs"), "--limit", 20)
    assert "wrote 20x6 id rows" in p.stdout
    r.ref_save_ivecs(ids[:20], os.path.join(tmp, "c.ivecs"))
    assert _bytes(os.path.join(tmp, "b.ivecs")) == _bytes(os.path.join(tmp, "c.ivecs"))


@needs_ref
def test_eval_recall_and_graph_accuracy(tmp):
    r = O.load("reference")
    rng = np.random.default_rng(3)
    gt = np.stack([rng.permutation(500)[:12] for _ in range(40)]).astype(np.uint32)
    res = gt[:, :10].copy()
    res[::3, 5:] = 499 - res[::3, 5:]  # some misses
    r.ref_save_ivecs(gt, os.path.join(tmp, "gt.ivecs"))
    r.ref_save_ivecs(res, os.path.join(tmp, "res.ivecs"))
    rec = np.mean([len(np.intersect1d(res[i], gt[i, :10])) / 10 for i in range(40)])
    p = run("eval", "--results", os.path.join(tmp, "res.ivecs"), "--gt", os.path.join(tmp, "gt.ivecs"),
            "--csv", os.path.join(tmp, "e.csv"))
    assert csv_rows(p.stdout) == [["metric", "value"], ["avg_recall", g10(rec)]]
    assert open(os.path.join(tmp, "e.csv")).read() == p.stdout
    # graph accuracy: a wider truth is sliced to the graph width
    p = run("eval", "--graph", os.path.join(tmp, "res.ivecs"), "--gt", os.path.join(tmp, "gt.ivecs"))
    assert csv_rows(p.stdout) == [["metric", "value"], ["graph_accuracy", g10(rec)]]
    assert run("eval", ok=False).returncode == 2


@needs_ref
def test_forest_file_validation_errors(tmp):
    r = O.load("reference")
    x = r.gen_synthetic(400, 6, 2)
    r.ref_save_fvecs(r.vs(x), os.path.join(tmp, "b.fvecs"))
    fr = r.build_forest(r.vs(x), 2, 8, 2)
    good = os.path.join(tmp, "f.akf")
    r.ref_save_forest(fr, good)
    blob = bytearray(_bytes(good))
    bad = os.path.join(tmp, "bad.akf")
    with open(bad, "wb") as fh:
        fh.write(blob[:-3])  # truncated
    p = run("build-graph", "--base", os.path.join(tmp, "b.fvecs"), "--forest", bad, "--seed", 1,
            "--out", os.path.join(tmp, "g.ivecs"), ok=False)
    assert p.returncode == 1 and ("forest file" in p.stderr or "unexpected end of file" in p.stderr)
    blob[0:4] = b"XXXX"
    with open(bad, "wb") as fh:
        fh.write(blob)
    p = run("build-graph", "--base", os.path.join(tmp, "b.fvecs"), "--forest", bad, "--seed", 1,
            "--out", os.path.join(tmp, "g.ivecs"), ok=False)
    assert p.returncode == 1 and "not a forest file" in p.stderr


# ------------------------------------------------------------------ GPU

@needs_ref
@pytest.mark.gpu
def test_cli_pipeline_matches_reference(tmp):
    """convert -> build-trees -> gt -> build-graph -> search -> eval, each
    artifact checked against the reference library's own output."""
    r = O.load("reference")
    n, nq, dim, trees, leaf, seed, k = 2000, 60, 16, 4, 8, 5, 10
    f = lambda name: os.path.join(tmp, name)
    run("convert", "--synthetic", f"{n}:{dim}:{seed}", "--out", f("base.fvecs"))
    run("convert", "--synthetic", f"{nq}:{dim}:{seed + 100}", "--out", f("q.fvecs"))
    x, q = r.gen_synthetic(n, dim, seed), r.gen_synthetic(nq, dim, seed + 100)
    vx, vq = r.vs(x), r.vs(q)

    # build-trees: AKF1 bytes
    p = run("build-trees", "--base", f("base.fvecs"), "--trees", trees, "--leaf-cap", leaf, "--seed", seed,
            "--workers", 8, "--out", f("f.akf"))
    assert f"tree build: n={n} dim={dim} trees={trees} leaf_cap={leaf} seed={seed}" in p.stdout
    fr = r.build_forest(vx, trees, leaf, seed)
    r.ref_save_forest(fr, f("ref.akf"))
    assert _bytes(f("f.akf")) == _bytes(f("ref.akf"))

    # gt: self mode with distances, query mode
    p = run("gt", "--base", f("base.fvecs"), "--k", 20, "--out", f("gt.ivecs"), "--out-dists", f("gt.fvecs"))
    gids, gd, comps = r.brute_force(vx, None, 20, with_dists=True)
    assert f"ground truth: k=20 mode=self dist_comps={comps}" in p.stdout
    r.ref_save_ivecs(gids, f("rgt.ivecs"))
    r.ref_save_fvecs(r.vs(gd), f("rgt.fvecs"))
    assert _bytes(f("gt.ivecs")) == _bytes(f("rgt.ivecs"))
    assert _bytes(f("gt.fvecs")) == _bytes(f("rgt.fvecs"))
    run("gt", "--base", f("base.fvecs"), "--queries", f("q.fvecs"), "--k", k, "--out", f("qgt.ivecs"))
    qgt = r.brute_force(vx, vq, k)
    r.ref_save_ivecs(qgt, f("rqgt.ivecs"))
    assert _bytes(f("qgt.ivecs")) == _bytes(f("rqgt.ivecs"))

    # build-graph (efanna, per-iteration accuracy against the 20-wide truth sliced to k)
    p = run("build-graph", "--base", f("base.fvecs"), "--forest", f("f.akf"), "--gt", f("gt.ivecs"), "--k", k,
            "--dep", 4, "--pool", 30, "--sample", 10, "--iters", 5, "--min-change-rate", 0, "--seed", seed,
            "--out", f("g.ivecs"), "--out-dists", f("g.fvecs"), "--log", f("g.csv"))
    # every logged column but the wall-clock seconds equals the reference's, `changes` included
    ids, dists, log, summ = r.build_graph(vx, fr, k=k, conquer_depth=4, pool_cap=30, sample_cap=10, max_iters=5,
                                          strategy=0, seed=seed, min_change_rate=0.0, gt=gids[:, :k])
    r.ref_save_ivecs(ids, f("rg.ivecs"))
    r.ref_save_fvecs(r.vs(dists), f("rg.fvecs"))
    assert _bytes(f("g.ivecs")) == _bytes(f("rg.ivecs"))
    assert _bytes(f("g.fvecs")) == _bytes(f("rg.fvecs"))
    rows = csv_rows(open(f("g.csv")).read())
    assert rows[0] == ["iteration", "seconds", "dist_comps", "changes", "accuracy"]
    assert len(rows) - 1 == len(log)
    for row, lg in zip(rows[1:], log):
        assert row[0] == str(int(lg[0])) and row[2] == str(int(lg[2])) and row[4] == g10(lg[4])
        assert row[3] == str(int(lg[3]))
    assert "# strategy=efanna" in open(f("g.csv")).read()

    # search: sweep, results of the last point, CSV averages
    p = run("search", "--base", f("base.fvecs"), "--queries", f("q.fvecs"), "--forest", f("f.akf"),
            "--graph", f("g.ivecs"), "--gt", f("qgt.ivecs"), "--k", k, "--seed", 9, "--sweep", "8:20,20:40",
            "--out", f("res.ivecs"), "--csv", f("s.csv"), "--per-query", f("pq.csv"))
    srows = csv_rows(open(f("s.csv")).read())
    assert srows[0] == ["expansion", "pool_size", "mean_time_us", "avg_dist_comps", "avg_seed_points", "avg_recall"]
    for row, (E, P) in zip(srows[1:], [(8, 20), (20, 40)]):
        rid, _, rst = r.search(vx, fr, ids, vq, k_return=k, pool_size=P, expansion=E, iters=4, seed=9)
        rec = np.mean([len(np.intersect1d(rid[i], qgt[i])) / k for i in range(nq)])
        assert row[:2] == [str(E), str(P)]
        assert row[3] == g10(rst[:, 0].astype(np.float64).sum() / nq)
        assert row[4] == g10(rst[:, 3].astype(np.float64).sum() / nq)
        assert row[5] == g10(rec)
    r.ref_save_ivecs(rid, f("rres.ivecs"))
    assert _bytes(f("res.ivecs")) == _bytes(f("rres.ivecs"))
    pq = csv_rows(open(f("pq.csv")).read())
    assert len(pq) == nq + 1 and [int(row[2]) for row in pq[1:]] == rst[:, 0].tolist()

    # random-init search writes the reference's results too
    run("search", "--base", f("base.fvecs"), "--queries", f("q.fvecs"), "--graph", f("g.ivecs"), "--k", k,
        "--random-init", "--seed", 9, "--sweep", "20:40", "--out", f("rr.ivecs"))
    rid2, _, _ = r.search(vx, None, ids, vq, k_return=k, pool_size=40, expansion=20, iters=4, seed=9,
                          random_init=True)
    r.ref_save_ivecs(rid2, f("rrr.ivecs"))
    assert _bytes(f("rr.ivecs")) == _bytes(f("rrr.ivecs"))

    # eval --k-list (accuracy vs k, eval.cpp:129-155)
    p = run("eval", "--graph", f("g.ivecs"), "--base", f("base.fvecs"), "--k-list", "1,5,10")
    want = r.ref_accuracy_vs_k(vx, ids, [1, 5, 10])
    assert csv_rows(p.stdout) == [["k", "accuracy"]] + [[str(kk), g10(a)] for kk, a in zip([1, 5, 10], want)]
