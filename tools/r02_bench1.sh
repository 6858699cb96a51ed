# 1-GPU bench + smoke of the current tree
O=gpurun_out/${1:-b1}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/rc.txt
for r in 1 2; do timeout 900 python bench.py > $O/bench$r.json 2> $O/bench$r.err; echo bench$r=$? >> $O/rc.txt; done
cat $O/rc.txt
