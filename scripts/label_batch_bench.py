"""label_batch over N TRJL files of 200 records (C8 shape): host ingestion +
GPU labelling wall time.  Usage: python scripts/label_batch_bench.py [N]"""
import os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_13211_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
script = P.EventScript(P.SubtaskKind.Pick, [P.ScriptStep(P.EventKind.Contact, 60),
                                            P.ScriptStep(P.EventKind.Grasped, 60),
                                            P.ScriptStep(P.EventKind.Success, 60)], tail=19)
trajs = P.realize_many([script] * n, list(range(n)))
with tempfile.TemporaryDirectory() as d:
    paths = []
    for i, t in enumerate(trajs):
        t.header.episode_id = f"ep-{i:06d}"
        pth = os.path.join(d, f"{i:06d}.trjl")
        P.write_binary_file(t, pth)
        paths.append(pth)
    P.label_batch(paths[:10])
    t0 = time.perf_counter()
    res = P.label_batch(paths)
    dt = time.perf_counter() - t0
    print(f"label_batch {n} files x 200 records: {dt:.3f} s, {len(res.labels)} labels, "
          f"{len(res.errors)} errors, modes {res.mode_counts}")
