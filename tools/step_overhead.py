"""Times build steps under different harness settings (profiler, clock sampler)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

cfg = dict(bench.CONFIGS["cfg2"])
base, queries = bench.gen_data(cfg)
vs = A.VectorSet(base)
f = A.build_forest(vs, cfg["trees"], cfg["leaf"], bench.SEED)


def step():
    s = A.init_graph(vs, f, cfg["k"], cfg["dep"], cfg["P"], cfg["S"], bench.SEED)
    t = [time.perf_counter()]
    for _ in range(2):
        A.detail.nn_descent_iteration(s, vs)
        t.append(time.perf_counter())
    return s, t


for mode in ["plain", "plain", "prof", "sampler", "prof+sampler", "plain"]:
    A.profile_reset()
    A.profile_enable("prof" in mode)
    clk = bench.ClockSampler(0) if "sampler" in mode else None
    if clk:
        clk.__enter__()
        time.sleep(0.5)
    t0 = time.perf_counter()
    s, ts = step()
    t1 = time.perf_counter()
    if clk:
        clk.__exit__(None, None, None)
    A.profile_enable(False)
    rep = A.profile_report()
    print(mode, f"total {t1 - t0:.3f}s init {ts[0] - t0:.3f} it1 {ts[1] - ts[0]:.3f} it2 {ts[2] - ts[1]:.3f}",
          f"kernels {sum(v[1] for v in rep.values()) / 1e3:.3f}s", flush=True)
    del s

# per-kernel breakdown of one step, per phase
for phase in ("init", "it1", "it2", "it3"):
    pass
A.profile_reset()
A.profile_enable(True)
s = A.init_graph(vs, f, cfg["k"], cfg["dep"], cfg["P"], cfg["S"], bench.SEED)
rep0 = A.profile_report()
print("init:", {k: round(v[1], 2) for k, v in rep0.items()})
for it in range(3):
    A.profile_reset()
    A.detail.nn_descent_iteration(s, vs)
    rep = A.profile_report()
    print(f"it{it + 1}:", {k: round(v[1], 2) for k, v in sorted(rep.items(), key=lambda kv: -kv[1][1])}, A.state_stats(s), s.meta()["dist_comps"])
A.profile_enable(False)
