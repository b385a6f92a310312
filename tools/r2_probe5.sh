set -u
export PYTHONPATH=$PWD
O=gpurun_out/p5; mkdir -p $O
free -g > $O/free.txt; nproc >> $O/free.txt; df -h /tmp >> $O/free.txt
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 600 python tools/probe_dense.py supremacy 30 --eb 1e-7 --reps 2 --kprof > $O/sup30.log 2>&1
timeout 600 python tools/probe_dense.py qft 30 --m 20 --eb 1e-5 --reps 2 > $O/qft30m20.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_enc_lossy --launch-skip 1 --launch-count 1 \
   -o $O/enc_sup30 -f python tools/probe_dense.py supremacy 30 --eb 1e-7 --reps 1 > $O/ncu_enc.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo probe-done
