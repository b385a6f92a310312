#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/f7; mkdir -p $O
( time python bench.py ) > $O/bench.json 2> $O/bench.err
( time python bench.py --impl reference --steps 10 --warmup 3 ) > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-companions > $O/ncu_list.log 2>&1
(rm -rf build/obj paper_2309_16979_b200/lib && python -c "import __graft_entry__ as g; g.build(); g.smoke()") > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
echo done
