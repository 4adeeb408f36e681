for t in 0 6000000 2000000 600000 200000 20000; do
  AMGR_TAIL_NNZ=$t ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv --log-file gpurun_out/tail_sweep_$t.csv python tools/region_driver.py 256 vcycle > /dev/null 2>&1
done
echo done
