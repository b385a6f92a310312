#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/f2; mkdir -p $O
python -m pytest tests/test_gpu_fresh.py -q > $O/fresh_tests.log 2>&1; echo "rc=$?" >> $O/fresh_tests.log
( time python bench.py ) > $O/bench.json 2> $O/bench.err
