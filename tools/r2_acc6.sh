#!/bin/bash
# reference acceptance criterion 6 (pipelining overlap) repeated + the GPU suite
export LD_LIBRARY_PATH=$PWD/paper_2309_16979_b200/lib
O=gpurun_out/acc6b; mkdir -p $O
for i in 1 2 3 4 5 6 7 8; do (cd /tmp && $OLDPWD/build/reftests/acceptance 6) >> $O/acc6.log 2>&1; done
export PYTHONPATH=$PWD
python -m pytest tests -m gpu -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
