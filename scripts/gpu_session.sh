#!/bin/bash
# One GPU session under gpurun: GPU tests, smoke, bench, optional ncu.  Usage:
#   gpurun --timeout S -- 'bash scripts/gpu_session.sh TAG "tests|smoke|bench|ncu|kb" [bench args]'
TAG=${1:-s}; WHAT=${2:-"tests smoke bench"}; shift 2; BARGS="$@"
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $O/smi.txt 2>&1
for w in $WHAT; do
  case $w in
    tests) timeout 2400 python -m pytest tests -m gpu -q -rA --durations=40 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt ;;
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt ;;
    bench) timeout 1800 python bench.py $BARGS > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/rc.txt ;;
    kb) timeout 900 python scripts/kernel_bench.py > $O/kb.json 2> $O/kb.err; echo "kb rc=$?" >> $O/rc.txt ;;
    ncu) timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 40 --warmup 0 --no-cpu-baseline --profile-leaves 4 > $O/ncu_bench.log 2>&1; echo "ncu-list rc=$?" >> $O/rc.txt
         timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 40 -c 1 -o $O/k_fused_full python bench.py --steps 40 --warmup 0 --no-cpu-baseline --profile-leaves 4 > $O/ncu_full.log 2>&1; echo "ncu-full rc=$?" >> $O/rc.txt ;;
  esac
done
tail -5 $O/pytest.log 2>/dev/null; cat $O/rc.txt; tail -c 3000 $O/bench.log 2>/dev/null
