set -u
export PYTHONPATH=$PWD
O=gpurun_out/ceil3; mkdir -p $O
timeout 900 python tools/run_large.py --circuit qft --n 36 --m 30 --eb 1e-5 --residency hbm > $O/qft36_hbm.json 2> $O/qft36.err
timeout 900 python tools/run_large.py --circuit ghz --n 38 --m 30 --eb 1e-5 --residency hbm > $O/ghz38_hbm.json 2> $O/ghz38.err
timeout 1500 python tools/run_large.py --circuit qft --n 38 --m 30 --eb 1e-5 --residency hbm > $O/qft38_hbm.json 2> $O/qft38.err
timeout 1500 python tools/run_large.py --circuit supremacy --n 34 --m 30 --eb 1e-7 --residency host > $O/sup34_host.json 2> $O/sup34_host.err
timeout 1500 python tools/run_large.py --circuit supremacy --n 34 --m 30 --eb 1e-7 --residency hbm > $O/sup34_hbm.json 2> $O/sup34_hbm.err
echo done
