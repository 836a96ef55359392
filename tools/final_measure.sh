#!/bin/bash
# Round-end measurements on a B200 box (run through gpurun from the repo
# root): GPU tests, the two bench arms, the ncu launch list of the bench, ncu
# --set full captures of the hot kernels, the DRAM traffic per launch class,
# the BASELINE matrix and the generic-path cliff.  Outputs in gpurun_out/.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/final_gputest.log 2>&1
echo "pytest rc $?" >> $O/final_gputest.log
timeout 600 python bench.py > $O/final_bench.json 2> $O/final_bench.err
echo "bench rc $?"
timeout 600 python bench.py --impl reference > $O/final_bench_reference.json 2>> $O/final_bench.err
echo "reference rc $?"
# launch list of the same command as the bench (durations are serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file $O/final_launches.csv python bench.py --steps 1 --warmup 1 \
  --no-cpu-baseline --eps-sweep > $O/final_ncu_launches.log 2>&1
# DRAM traffic per launch class (3 frames)
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none --csv --log-file $O/final_traffic.csv \
  python tools/ncu_frame.py 5 3 1e-3 > $O/final_ncu_traffic.log 2>&1
# full captures of the hot kernels (frame 1 of a 3-frame run)
for k in enc_block_kernel bs_chain_kernel bs_interior_kernel dec_block_fast_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k \
    --launch-skip 1 -c 1 -f -o $O/final_$k python tools/ncu_frame.py 5 3 1e-3 \
    > $O/final_ncu_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"bs_interior_kernelILb0|bs_interior_kernel<0" --launch-skip 1 -c 1 -f \
  -o $O/final_bs_interior_dec python tools/ncu_frame.py 5 3 1e-3 > $O/final_ncu_intdec.log 2>&1
timeout 900 python bench.py --matrix $O/final_matrix.json > $O/final_matrix.log 2>&1
timeout 900 python tools/cliff_time.py > $O/final_cliff.json 2> $O/final_cliff.err
ls -la $O | tail -30
