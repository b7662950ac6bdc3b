#!/bin/bash
# SASS opcode evidence per object of libsped.so (tcgen05 MMA / TMEM loads /
# bulk copies / 256-bit gathers).  usage: tools/sass_histogram.sh > profiles/rNN_sass_histogram.txt
cd "$(dirname "$0")/../build/sped" || exit 1
ops="UTCHMMA UTCBAR LDTM UBLKCP UTMALDG LDG.E.ENL2.256 LDG.E.128 LDG.E.64 STG.E.128 SYNCS"
printf "%-12s" object; for m in $ops; do printf " %15s" $m; done; echo
for o in *.o; do
  [[ $o == *_* && $o != edge_batch.o && $o != csr_build.o && $o != gram_tc.o && $o != update_tc.o ]] && continue
  s=$(cuobjdump -sass "$o" 2>/dev/null)
  printf "%-12s" "${o%.o}"
  for m in $ops; do printf " %15s" "$(grep -c -- "$m" <<<"$s")"; done; echo
done
