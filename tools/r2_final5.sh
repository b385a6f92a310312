#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/f5; mkdir -p $O
( time python bench.py ) > $O/bench.json 2> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-companions > $O/ncu_list.log 2>&1
echo done
