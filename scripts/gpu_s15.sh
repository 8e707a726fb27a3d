O=gpurun_out/s15; mkdir -p $O
for i in 1 2; do
timeout 300 python scripts/repro_range.py C3 128 0 147 188 > $O/rel_$i.txt 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/repro_range.py C3 128 0 147 188 > $O/rel_blk_$i.txt 2>&1
TUSQ_LIB_NAME=libtusq_dbg.so timeout 300 python scripts/repro_range.py C3 128 0 147 188 > $O/dbg_$i.txt 2>&1
done
for f in $O/*.txt; do echo $f; tail -n 2 $f; done
