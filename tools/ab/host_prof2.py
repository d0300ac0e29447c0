import cProfile, pstats, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1811_11629_b200 as R
p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
out = torch.empty(1 << 20, dtype=torch.float64, device="cuda")
for mv in (1, 65536):
    st = R.init_vector(p, mv=mv)
    for _ in range(20): R.take_floats(st, 1 << 20, out=out)
    torch.cuda.synchronize()
    pr = cProfile.Profile(); pr.enable()
    for _ in range(500): R.take_floats(st, 1 << 20, out=out)
    pr.disable(); torch.cuda.synchronize()
    print("==== mv", mv)
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
