set -u
export PYTHONPATH=$PWD
O=gpurun_out/p4; mkdir -p $O
timeout 600 python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 2 --kprof > $O/sup30m28.log 2>&1
timeout 600 python tools/probe_dense.py qft 30 --m 20 --eb 1e-5 --reps 2 --kprof > $O/qft30m20.log 2>&1
timeout 600 python tools/probe_dense.py supremacy 30 --eb 1e-7 --reps 2 --kprof > $O/sup30.log 2>&1
echo probe-done
