set -u
export PYTHONPATH=$PWD
O=gpurun_out/p8; mkdir -p $O
timeout 300 python tools/probe_dense.py qft 30 --m 30 --eb 1e-5 --reps 3 --kprof > $O/qft30.log 2>&1
QZ_NO_WMAP=1 timeout 300 python tools/probe_dense.py qft 30 --m 30 --eb 1e-5 --reps 3 --kprof > $O/qft30_nowmap.log 2>&1
timeout 300 python tools/probe_dense.py supremacy 30 --m 30 --eb 1e-7 --reps 2 --kprof > $O/sup30.log 2>&1
QZ_NO_WMAP=1 timeout 300 python tools/probe_dense.py supremacy 30 --m 30 --eb 1e-7 --reps 2 --kprof > $O/sup30_nowmap.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tile_pass_reg --launch-skip 3 --launch-count 1 \
   -o $O/pass4_qft30 -f python tools/probe_timing.py qft relaxed > $O/ncu_pass.log 2>&1
echo probe-done
