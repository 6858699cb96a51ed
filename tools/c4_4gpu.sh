# C4 strong scaling at N GPUs repeated (variance check), then C2 weak once
O=gpurun_out/${C4_TAG:-c4rep}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
N=${1:-4}
for r in 1 2 3; do timeout 900 python bench.py --gpus $N --config C4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c4_$r.json 2> $O/bench_c4_$r.err; echo bench_c4_$r=$? >> $O/rc.txt; done
timeout 900 python bench.py --gpus $N > $O/bench_c2.json 2> $O/bench_c2.err; echo bench_c2=$? >> $O/rc.txt
cat $O/rc.txt
