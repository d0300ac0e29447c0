#!/bin/bash
# Offline SASS A/B: compile fill.cu with extra -D flags and print the heavy
# slots / ALU ops / instructions per draw of the fast fill loop for each e.
#   tools/ab/sass_ab.sh -DRSA_MSG_VARIANT=1
set -e
cd "$(dirname "$0")/../.."
out=/tmp/sass_ab_$$.cubin
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -Iinclude "$@" -cubin -o $out paper_1811_11629_b200/csrc/fill.cu
for e in 3 9 65537; do
  cuobjdump -sass -fun "_ZN3rsa11k_fill_fastILj${e}ELi2ELb0ELi1EEEvPK12rsa_instancejmmPmS4_S4_S4_Pdmj" $out 2>/dev/null \
    | grep -E "/\*[0-9a-f]{4}\*/" > /tmp/sass_ab_$$.txt
  echo "e=$e $(python tools/sass_slots.py /tmp/sass_ab_$$.txt --lightest 2>/dev/null | head -1)"
done
rm -f $out /tmp/sass_ab_$$.txt
