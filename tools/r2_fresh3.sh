#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/f3; mkdir -p $O
python -m pytest tests/test_gpu_fresh.py -q > $O/fresh_tests.log 2>&1; echo "rc=$?" >> $O/fresh_tests.log
python -m pytest tests -m gpu -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
