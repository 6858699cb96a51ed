# Round-2 GPU check (run under gpurun from the repo root): loopback multi-rank
# tests first (new), then the whole GPU suite, smoke and a short bench.
O=gpurun_out/${1:-r02a}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.max.mem,power.limit --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$? >> $O/rc.txt
timeout 900 python -m pytest tests/test_loopback.py -m gpu -x -q -s --durations=5 > $O/loopback.log 2>&1; echo loopback=$? >> $O/rc.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > $O/gpu_tests.log 2>&1; echo tests=$? >> $O/rc.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/rc.txt
timeout 900 python bench.py > $O/bench1.json 2> $O/bench1.err; echo bench1=$? >> $O/rc.txt
cat $O/rc.txt
