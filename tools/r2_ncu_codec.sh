#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/nc2; mkdir -p $O
python -m pytest tests/test_gpu_codec.py -q -x > $O/codec_tests.log 2>&1; echo "rc=$?" >> $O/codec_tests.log
python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 2 --kprof > $O/sup_m28.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_enc_lossy --launch-count 3 \
   -o $O/sup_encode -f python tools/probe_dense.py supremacy 30 --c 16 --m 30 --eb 1e-7 --reps 1 > $O/ncu_enc.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dec_lossy_seg --launch-skip 2 --launch-count 1 \
   -o $O/sup_decode -f python tools/probe_dense.py supremacy 30 --m 28 --depth 8 --eb 1e-7 --reps 1 > $O/ncu_dec.log 2>&1
echo done
