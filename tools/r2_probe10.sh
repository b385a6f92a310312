set -u
export PYTHONPATH=$PWD
O=gpurun_out/p10; mkdir -p $O
QZ_DEBUG_COUNTERS=1 timeout 300 python tools/probe_dense.py supremacy 30 --m 30 --eb 1e-7 --reps 1 > $O/sup30_counters.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tile_pass_reg --launch-skip 20 --launch-count 1 \
   -o $O/sup_pass20 -f python tools/probe_dense.py supremacy 30 --m 30 --eb 1e-7 --reps 1 > $O/ncu_sup.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tile_pass_reg --launch-skip 3 --launch-count 1 \
   -o $O/sup_pass3 -f python tools/probe_dense.py supremacy 30 --m 30 --eb 1e-7 --reps 1 > $O/ncu_sup3.log 2>&1
echo probe-done
