"""Times atkg_simulate_recall_many (GPU top-k) vs the reference's simulate_recall_many (CPU)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_04165_b200 as atk  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from tests.test_simulate import ref_simulate  # noqa: E402

threads = os.cpu_count()
for n, runs in [(1 << 16, 1024), (1 << 20, 256)]:
    cfgs = [atk.AlgoParams(n=n, num_buckets=b, local_k=kp, global_k=k)
            for b, kp, k in [(256, 1, 64), (256, 2, 64), (512, 4, 256)]]
    atk.simulate_recall_many(cfgs, 8, 1, threads=threads)
    t = time.perf_counter(); ours = atk.simulate_recall_many(cfgs, runs, 1, threads=threads); t1 = time.perf_counter() - t
    os.environ["ATKG_SIM_HOST_GEN"] = "1"
    t = time.perf_counter(); hostgen = atk.simulate_recall_many(cfgs, runs, 1, threads=threads); t3 = time.perf_counter() - t
    del os.environ["ATKG_SIM_HOST_GEN"]
    t = time.perf_counter(); mean, sd = ref_simulate(O.ref().lib, cfgs, runs, 1, threads=threads); t2 = time.perf_counter() - t
    same = all(h.mean_recall == m for h, m in zip(hostgen, mean)) and all(o.mean_recall == m and o.stddev == s for o, m, s in zip(ours, mean, sd))
    print(f"n={n} runs={runs} configs=3 threads={threads}: ours {t1:.3f} s (host-generated rows {t3:.3f} s), reference {t2:.3f} s, "
          f"identical={same}, recall={[round(o.mean_recall, 4) for o in ours]}")
