#!/bin/bash
# usage: scripts/sweep.sh "<case>" "ENV1=.. ENV2=.." "ENV..." ...
# times each env config and collects DRAM bytes of the star kernel with ncu
case_="$1"; shift
for cfg in "$@"; do
  t=$(env $cfg timeout 120 python scripts/quick_time.py $case_ 2>&1 | tail -1)
  m=$(env $cfg timeout 120 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:star3 -s 2 -c 2 python scripts/quick_time.py $case_ 2>/dev/null | grep -E "dram__bytes|gpu__time|hit_rate" | awk '{print $1"="$(NF)}' | tr '\n' ' ')
  echo "[$cfg] $t | $m"
done
