#!/usr/bin/env bash
# ncu --set full of the vector-path kernels at their best blocks (and the
# scalar TMA kernel beside them); digests + raw + source pages.
cd "$(dirname "$0")/.."
O=gpurun_out/${OUT:-r02e}; mkdir -p $O
cap() { # name kernel-regex args...
  local n=$1 k=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/$n python scripts/profile_pass.py "$@" > $O/$n.log 2>&1
  python scripts/ncu_digest.py $O/$n.ncu-rep > $O/${n}_digest.txt 2>/dev/null
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/${n}_raw.csv 2>/dev/null
  ncu -i $O/$n.ncu-rep --page source --csv > $O/${n}_source.csv 2>/dev/null
  rm -f $O/$n.ncu-rep
}
for spec in "$@"; do
  set -- $spec
  cap "$@"
done
ls $O
