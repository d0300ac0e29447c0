timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -c 1 -o gpurun_out/prof_c3 -f python bench.py --config 3 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_c3.log 2>&1; tail -1 gpurun_out/ncu_c3.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_seg_ -c 4 -o gpurun_out/prof_seg -f python -c "
import torch, paper_1811_11629_b200 as R
p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
st = R.init_vector(p, mv=1)
out = torch.empty(1 << 20, dtype=torch.float64, device='cuda')
R.take_floats(st, 1 << 20, out=out); torch.cuda.synchronize()" > gpurun_out/ncu_seg.log 2>&1; tail -1 gpurun_out/ncu_seg.log
