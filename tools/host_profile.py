import cProfile, pstats, time, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1811_11629_b200 as R
p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
st = R.init_vector(p, mv=1)
out = torch.empty(1 << 20, dtype=torch.float64, device="cuda")
for _ in range(20): R.take_floats(st, 1 << 20, out=out)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(200): R.take_floats(st, 1 << 20, out=out)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
