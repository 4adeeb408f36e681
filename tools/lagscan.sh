for L in 1 2 4 8; do echo "LAG=$L"; AMGR_LAG_ROUNDS=$L COARSE=exact timeout 300 python tools/vcycle_time.py 256 AMGR_LAG_FUSE 1 2>&1 | tail -1; done
