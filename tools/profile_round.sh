#!/bin/bash
# Round profiling recipe (run under gpurun): launch list of one V-cycle region
# and full captures of the dominant level-0 kernels at 256^3.
set -x
mkdir -p gpurun_out
python tools/region_driver.py 256 all > gpurun_out/plain_all.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/launches_all.csv python tools/region_driver.py 256 all > gpurun_out/ncu_list.log 2>&1
# rowpass launches in the region (rebuild has none): V-cycle 1 = 14 down + 14 smooth
python tools/region_driver.py 256 vcycle > gpurun_out/plain_v.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:k_rowpass -s 27 -c 1 -o gpurun_out/smooth_L0 python tools/region_driver.py 256 vcycle > gpurun_out/ncu_s.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:k_rowpass -s 0 -c 1 -o gpurun_out/down_L0 python tools/region_driver.py 256 vcycle > gpurun_out/ncu_d.log 2>&1
python tools/region_driver.py 256 rebuild > gpurun_out/plain_r.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:k_rap -s 0 -c 1 -o gpurun_out/rap_L0 python tools/region_driver.py 256 rebuild > gpurun_out/ncu_r.log 2>&1
tail -2 gpurun_out/ncu_*.log
