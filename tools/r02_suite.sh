# GPU suite + smoke of the current tree (one GPU)
O=gpurun_out/${1:-suite}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests=$? >> $O/rc.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/rc.txt
cat $O/rc.txt
