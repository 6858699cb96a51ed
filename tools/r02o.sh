O=gpurun_out/r02o
mkdir -p $O
for v in base sp2 sp3 sp2all sp2ku1 sp2ku3; do
  if [ $v = base ]; then L=""; else L=paper_2107_01243_b200/_var/libsem_$v.so; fi
  AX_ONLY=1 SEM_LIB=$L timeout 600 python tools/ax_ab.py M5,M6,M7,M8,M9,M10,M11 >> $O/ab.jsonl 2>> $O/ab.err
done
