O=gpurun_out/r02m
mkdir -p $O
for rep in 1 2; do
  timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab.jsonl 2>&1
  PCG_FUSE=0 timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab.jsonl 2>&1
  for v in pf41 pf51 pf22 pf34 pf42; do
    SEM_LIB=paper_2107_01243_b200/_var/libsem_$v.so timeout 300 python tools/ax_ab.py C2,C3 >> $O/ab.jsonl 2>&1
  done
done
SEM_LIB=paper_2107_01243_b200/_var/libsem_checked.so timeout 1800 python -m pytest tests -m gpu -q > $O/checked_tests.log 2>&1; echo checked=$? >> $O/rc.txt
