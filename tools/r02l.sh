O=gpurun_out/r02l
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fused_p_update or pcg_graph or pcg_parity or c3_fixed or helm or single_reduction" > $O/tests.log 2>&1; echo tests=$? >> $O/rc.txt
for rep in 1 2; do
  timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab.jsonl 2>&1
  PCG_FUSE=0 timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab.jsonl 2>&1
done
SEM_LIB=paper_2107_01243_b200/_var/libsem_checked.so timeout 1800 python -m pytest tests -m gpu -q -x > $O/checked_tests.log 2>&1; echo checked=$? >> $O/rc.txt
SEM_LIB=paper_2107_01243_b200/_var/libsem_checked.so timeout 600 python tools/sanitize_workload.py > $O/checked_workload.log 2>&1; echo checked_wl=$? >> $O/rc.txt
cat $O/rc.txt
