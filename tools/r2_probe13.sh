set -u
export PYTHONPATH=$PWD
O=gpurun_out/p13; mkdir -p $O
QZC_LIB=$PWD/paper_2309_16979_b200/lib_var/libqzcuda.so timeout 300 python tools/probe_dense.py qft 30 --m 30 --eb 1e-5 --reps 3 --kprof > $O/qft30_var.log 2>&1
QZC_LIB=$PWD/paper_2309_16979_b200/lib_var/libqzcuda.so timeout 300 python tools/probe_dense.py supremacy 30 --m 30 --eb 1e-7 --reps 1 > $O/sup30_var.log 2>&1
QZC_LIB=$PWD/paper_2309_16979_b200/lib_var/libqzcuda.so timeout 300 ncu --section LaunchStats --section Occupancy --clock-control none -k regex:tile_pass_reg --launch-skip 3 --launch-count 1 python tools/probe_timing.py qft relaxed > $O/ncu_occ_var.log 2>&1
timeout 300 ncu --section LaunchStats --section Occupancy --clock-control none -k regex:tile_pass_reg --launch-skip 3 --launch-count 1 python tools/probe_timing.py qft relaxed > $O/ncu_occ_base.log 2>&1
echo probe-done
