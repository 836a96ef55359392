#!/bin/bash
# Round-end measurements of the last session (kernels unchanged since
# final_measure.sh: no new --set full captures): GPU tests, the two bench
# arms, the ncu launch list of the bench command, DRAM traffic per class.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/final_gputest.log 2>&1
echo "pytest rc $?" >> $O/final_gputest.log
tail -n 3 $O/final_gputest.log
timeout 600 python bench.py > $O/final_bench.json 2> $O/final_bench.err
echo "bench rc $?"
timeout 600 python bench.py --impl reference > $O/final_bench_reference.json 2>> $O/final_bench.err
echo "reference rc $?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file $O/final_launches.csv python bench.py --steps 1 --warmup 1 \
  --no-cpu-baseline --eps-sweep > $O/final_ncu_launches.log 2>&1
echo "ncu launches rc $?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none --csv --log-file $O/final_traffic.csv \
  python tools/ncu_frame.py 5 3 1e-3 > $O/final_ncu_traffic.log 2>&1
echo "ncu traffic rc $?"
ls -la $O | tail -12
