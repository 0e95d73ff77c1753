"""Per NN-descent round at a bench config: changes (accepted inserts), offers
that beat the start-of-round tail, spilled offers, and per-kernel CUDA-event
times.  python tools/round_stats.py [cfg] [rounds]"""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"])
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 2
base, _ = bench.gen_data(cfg)
vs = A.VectorSet(base)
f = A.build_forest(vs, cfg["trees"], cfg["leaf"], bench.SEED)
for rep in range(2):
    A.profile_reset()
    A.profile_enable(True)
    s = A.init_graph(vs, f, cfg["k"], cfg["dep"], cfg["P"], cfg["S"], bench.SEED)
    for r in range(rounds):
        ch = A.detail.nn_descent_iteration(s, vs)
        st = A.state_stats(s)
        if rep:
            print(f"round {r + 1}: changes {ch:,} offers {st['offers']:,} ({ch / max(st['offers'], 1):.2f} accepted) "
                  f"join rows {st['join_rows']:,} spilled {st['spilled']:,} slots/pt {st['offer_slots']}")
    A.profile_enable(False)
    if rep:
        for name, (cnt, ms) in sorted(A.profile_report().items(), key=lambda kv: -kv[1][1])[:14]:
            print(f"    {name:30s} {cnt:4d} {ms:9.3f} ms")
    del s
