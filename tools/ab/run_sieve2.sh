for v in m6r16 m8r8 m8r16 m8r32; do
echo "== $v"
RSARAND_B200_LIB=tools/ab/lib_$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_scan_sieve -c 3 python -c "
from paper_1811_11629_b200 import paramfactory
paramfactory.safe_primes_u32(1 << 31, 1 << 32)" 2>&1 | grep -E "gpu__time" 
done
