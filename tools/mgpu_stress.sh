# stability at N GPUs: the parity worker twice and the bench five times (gpurun --gpus N)
O=gpurun_out/${ST_TAG:-stress}
mkdir -p $O
N=${1:-4}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for r in 1 2; do timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -s > $O/tests$r.log 2>&1; echo tests$r=$? >> $O/rc.txt; done
for r in 1 2 3 4 5; do timeout 600 python bench.py --gpus $N --no-e2e --no-cpu-baseline --steps 200 > $O/bench$r.json 2> $O/bench$r.err; echo bench$r=$? >> $O/rc.txt; done
cat $O/rc.txt
