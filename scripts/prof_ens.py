"""cProfile of one run_ensemble call (ens workload) after warm-up: where the host time goes."""
import cProfile, pstats, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_22092_b200 as fs
g = fs.gen_erdos_renyi(1000, 8.0, seed=20250809)
m = fs.seir_standard(0.25, 5.0, 4.0, 7.5, 5.0)
cfg = fs.RenewalConfig()
run = lambda: fs.run_ensemble("renewal", g, m, cfg, 20250809, 50.0, 100, seed_count=10)
for _ in range(3):
    run()
torch.cuda.synchronize()
t0 = time.perf_counter(); run(); torch.cuda.synchronize(); print("wall ms", round((time.perf_counter() - t0) * 1e3, 2))
pr = cProfile.Profile()
pr.enable(); run(); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
