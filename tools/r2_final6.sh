#!/bin/bash
# closing measurement: bench (default), launch list, ncu of the dominant pass, switch tests
export PYTHONPATH=$PWD
O=gpurun_out/f6; mkdir -p $O
( time python bench.py ) > $O/bench.json 2> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-companions > $O/ncu_list.log 2>&1
QZ_NO_WARMUP=1 QZ_JIT_SYNC=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:qz_jit_pass --launch-skip 9 --launch-count 1 \
   -o $O/qft_last -f python tools/probe_dense.py qft 30 --c 16 --m 30 --eb 1e-5 --reps 1 > $O/ncu.log 2>&1
python -m pytest tests/test_gpu_sim.py -q -k "switches" > $O/switch.log 2>&1; echo "rc=$?" >> $O/switch.log
echo done
