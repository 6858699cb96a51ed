# multi-GPU parity worker incl. the peer-memory failure path (gpurun --gpus N)
O=gpurun_out/${MT_TAG:-fp1}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -q -s > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
cat $O/rc.txt
