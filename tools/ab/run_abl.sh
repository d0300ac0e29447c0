cp paper_1811_11629_b200/librsarand_b200.so tools/ab/lib_cur.so
for v in cur abl_f abl_b abl_beta abl_all; do
 echo "== $v"; RSARAND_B200_LIB=tools/ab/lib_$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_setup -c 2 python -c "
import paper_1811_11629_b200 as R
for _ in range(2): R.derive_params_table(R.DEFAULT_MASTER_SEED, 0, 1 << 20, validate=False) if False else None
from paper_1811_11629_b200 import paramfactory
t = paramfactory.safe_prime_table()
cfg = paramfactory._setup_config(R.DEFAULT_MASTER_SEED, 0, 9, len(paramfactory.MULTIPLIER_TABLE), 0)
import torch
from paper_1811_11629_b200 import _lib, _device
n = 1 << 20
mult = t.mult_table(tuple(paramfactory.MULTIPLIER_TABLE))
inst = torch.empty((n, 128), dtype=torch.uint8, device='cuda'); st = torch.empty(n, dtype=torch.int32, device='cuda')
for _ in range(2):
    _lib.call('rsa_setup_instances', cfg, n, mult.data_ptr(), t.sp.data_ptr(), t.n_sp, t.index.data_ptr(), t.sp.data_ptr(), t.n_p1, inst.data_ptr(), st.data_ptr(), None, _device.stream(inst.device))
torch.cuda.synchronize()" 2>&1 | grep "gpu__time_duration" 
done
