O=gpurun_out/r02e
mkdir -p $O
for rep in 1 2; do
for v in base rev keep revkeep revkeep42; do
  SEM_LIB=paper_2107_01243_b200/_var/libsem_$v.so timeout 300 python tools/ax_ab.py C2,C3 >> $O/ax_ab.jsonl 2>> $O/ax_ab.err
done
done
echo done
