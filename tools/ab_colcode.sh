# A/B of the coded column stream (AMGR_COLCODE: 0 = int32 columns,
# default = uint8 codes on the <= 8 nnz/row levels, 16 = also uint16 codes)
for v in 0 default 16 0 default 16; do
  if [ "$v" = default ]; then unset AMGR_COLCODE; else export AMGR_COLCODE=$v; fi
  timeout 600 python bench.py --no-strategies --no-e2e > gpurun_out/cc_$v.json 2>gpurun_out/cc_$v.err
  python -c "import json;d=json.load(open('gpurun_out/cc_$v.json'));print('colcode','$v',round(d['value'],2),round(d['roofline']['frac'],3),round(d['phase_rooflines']['vcycle']['ms'],3),round(d['phase_rooflines']['bicgstab_iteration']['ms'],3),d['clocks']['sm_mhz'])"
done
unset AMGR_COLCODE
