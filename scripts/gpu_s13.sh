O=gpurun_out/s13; mkdir -p $O
for L in libtusq.so libtusq_b1.so libtusq_b2.so; do
  TUSQ_LIB_NAME=$L timeout 600 python scripts/repro_c3.py C3 > $O/repro_$L.txt 2>&1
done
CUDA_LAUNCH_BLOCKING=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/repro_c3.py C3 > $O/sanitizer.txt 2>&1
tail -n 5 $O/repro_*.txt; head -c 6000 $O/sanitizer.txt
