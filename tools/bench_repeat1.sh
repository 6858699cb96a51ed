# 1-GPU: bench three times (default flags) and the reference arm
O=gpurun_out/${BR_TAG:-brep1}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for r in 1 2 3; do timeout 900 python bench.py > $O/bench$r.json 2> $O/bench$r.err; echo bench$r=$? >> $O/rc.txt; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$? >> $O/rc.txt
cat $O/rc.txt
