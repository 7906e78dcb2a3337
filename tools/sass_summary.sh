#!/bin/bash
# SASS evidence per cubin of libhalo_b200.so: counts of the Blackwell
# tensor-core / TMEM / TMA instructions (B200_PROFILING.md mnemonics).
# Usage: bash tools/sass_summary.sh > profiles/sass_r02.txt   (no GPU needed)
set -e
SO=${1:-$(dirname "$0")/../paper_2501_02625_b200/libhalo_b200.so}
T=$(mktemp -d)
cd "$T"
cuobjdump -xelf all "$SO" > /dev/null
echo "# SASS instruction counts per cubin of $(basename "$SO") (cuobjdump -sass)"
printf "%-28s %8s %8s %8s %8s %8s %8s %8s %8s %8s %8s\n" cubin UTCIMMA UTCQMMA UTCBAR LDTM STTM UTMALDG UTMASTG UBLKCP SHFL FADD2
for c in *.cubin; do
  cuobjdump -sass "$c" > s.txt
  cnt() { grep -cE "$1" s.txt || true; }
  printf "%-28s %8s %8s %8s %8s %8s %8s %8s %8s %8s %8s\n" "${c%.sm_100a.cubin}" "$(cnt 'UTCIMMA')" "$(cnt 'UTCQMMA')" \
    "$(cnt 'UTCBAR')" "$(cnt 'LDTM')" "$(cnt 'STTM')" "$(cnt 'UTMALDG')" "$(cnt 'UTMASTG')" "$(cnt 'UBLKCP')" \
    "$(cnt 'SHFL')" "$(cnt 'FADD2')"
done
echo
echo "# variants of the tensor-core instructions in gemm_sm100"
cuobjdump -sass gemm_sm100.sm_100a.cubin | grep -oE "UTC[A-Z]+MMA[.A-Z0-9]*|UTCBAR[.A-Z0-9]*|UTMALDG[.A-Z0-9]*|UTMASTG[.A-Z0-9]*" | sort | uniq -c
rm -rf "$T"
