#!/bin/bash
export PYTHONPATH=$PWD
O=gpurun_out/f1; mkdir -p $O
( time python bench.py ) > $O/bench.json 2> $O/bench.err
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
