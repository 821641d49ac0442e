#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/s8i3.log
for i in 1 2 3 4 5 6 7 8 9 10; do
  TPS_WATCHDOG=40 TPS_DUMP_AFTER=60 timeout 75 python tools/profile_resnet.py --mb 16 --stages 8 --variant I --pool 4 > /tmp/o.txt 2>/tmp/e.txt
  rc=$?
  echo "run $i rc=$rc" >> gpurun_out/s8i3.log
  if [ $rc -ne 0 ]; then tail -40 /tmp/e.txt >> gpurun_out/s8i3.log; break; fi
done
