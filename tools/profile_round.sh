#!/bin/bash
# Round profiling recipe (run under gpurun, one GPU): the launch list of one
# region (rebuild + 2 V-cycles + 2 solve iterations) and --set full captures
# of the dominant kernels at 256^3; tools/ncu_summarize.py turns them into
# profiles/<round>_ncu_full_summary.json and <round>_traffic.json.
# Each ncu command runs only after the same command exited 0 without ncu.
R=${1:-r01}
mkdir -p gpurun_out
full() {  # full <name> <what> <regex> <skip>
  ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:"$3" -s $4 -c 1 -o gpurun_out/$1 python tools/region_driver.py 256 $2 > gpurun_out/ncu_$1.log 2>&1
}
python tools/region_driver.py 256 all > gpurun_out/plain_all.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/${R}_launches.csv python tools/region_driver.py 256 all > gpurun_out/ncu_list.log 2>&1
python tools/region_driver.py 256 vcycle > gpurun_out/plain_v.log 2>&1 && {
  # level 0 runs k_dia (symmetric-stencil form): down L0 (0), smooth L0 (1);
  # ^k_rowpass$ then carries down L1..L13 and up L13..L1
  full smooth_L0 vcycle '^k_dia$' 1
  full down_L0 vcycle '^k_dia$' 0
  full down_L1 vcycle '^k_rowpass$' 0
}
python tools/region_driver.py 256 rebuild > gpurun_out/plain_r.log 2>&1 && {
  full rap_L0 rebuild '^k_rap_grp$' 0
  full rap_L1 rebuild '^k_rap_grp$' 1
}
python tools/ncu_summarize.py $R
# (copy gpurun_out/${R}_launches.csv to profiles/${R}_launches_256_rebuild_vcycle_solve.csv)
tail -n 2 gpurun_out/ncu_*.log
