ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv python bench.py --config 1 --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_setup|k_sp_index" -c 2 -o gpurun_out/prof_setup2 -f python -c "
import paper_1811_11629_b200 as R
R.derive_params_table(R.DEFAULT_MASTER_SEED, 0, 1 << 20)" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pd_" -c 2 -o gpurun_out/prof_pd2 -f python -c "
import torch, paper_1811_11629_b200 as R
p = R.derive_stream_params(R.StreamKey(R.DEFAULT_MASTER_SEED, 0))
out = torch.empty(1 << 20, dtype=torch.float64, device='cuda')
st = R.init_vector(p, mv=1); R.take_floats(st, 1 << 20, out=out); torch.cuda.synchronize()" > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches_c1.csv
