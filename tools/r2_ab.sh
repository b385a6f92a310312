L=paper_2309_16979_b200/lib
for r in 1 2 3; do for v in old new; do
cp $L/libqzcuda.so.$v $L/libqzcuda.so
python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), round(d['e2e']['value']))"
done; done
cp $L/libqzcuda.so.new $L/libqzcuda.so
