O=gpurun_out/s9; mkdir -p $O
timeout 600 python scripts/k5_micro.py > $O/micro_default.txt 2>&1
TUSQ_LIB_NAME=libtusq_dbg.so TUSQ_DBG_IDENTITY=1 timeout 600 python scripts/k5_micro.py > $O/micro_identity.txt 2>&1
TUSQ_LIB_NAME=libtusq_dbg.so TUSQ_DBG_WCONTIG=1 timeout 600 python scripts/k5_micro.py > $O/micro_wcontig.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 3 -o $O/k5_full python scripts/c4_batch.py 2600 8 > $O/ncu_full.log 2>&1
tail -n 12 $O/micro_*.txt
