# bench five times at N GPUs (gpurun --gpus N)
O=gpurun_out/${BR_TAG:-brep}
mkdir -p $O
N=${1:-4}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for r in 1 2 3 4 5; do timeout 600 python bench.py --gpus $N --no-e2e --no-cpu-baseline > $O/bench$r.json 2> $O/bench$r.err; echo bench$r=$? >> $O/rc.txt; done
cat $O/rc.txt
