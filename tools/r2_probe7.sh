set -u
export PYTHONPATH=$PWD
O=gpurun_out/p7; mkdir -p $O
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_enc_lossy --launch-skip 1 --launch-count 1 \
   -o $O/enc_qft30 -f python tools/probe_timing.py qft relaxed > $O/ncu_enc_qft.log 2>&1
timeout 600 python tools/probe_timing.py qft relaxed > $O/qft30.log 2>&1
echo probe-done
