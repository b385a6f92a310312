#!/bin/bash
# Round profile capture on one B200 (run under gpurun from the repo root):
#   bench line (+ reference arm), ncu launch list of the same bench command,
#   one `ncu --set full` capture of the heaviest fused gate pass.
# Outputs land in gpurun_out/prof/; the summary is written by hand into
# profiles/rN_summary.md.
set -u
R=${1:-r1}
O=gpurun_out/prof
mkdir -p $O
export PYTHONPATH=$PWD
python bench.py --steps 3 --warmup 3 > $O/${R}_bench.log 2>&1 && tail -1 $O/${R}_bench.log > $O/${R}_bench.json
python bench.py --impl reference --steps 2 --warmup 1 > $O/${R}_ref.log 2>&1 && tail -1 $O/${R}_ref.log > $O/${R}_bench_reference.json
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/${R}_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
# heaviest QFT-30 pass: the 4th tile_pass_reg launch of a run
python tools/probe_timing.py qft relaxed > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tile_pass_reg --launch-skip 3 --launch-count 1 \
    -o $O/${R}_tile_pass_full -f python tools/probe_timing.py qft relaxed > $O/ncu_full.log 2>&1
echo done
