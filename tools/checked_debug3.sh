O=gpurun_out/${CD_TAG:-chkdbg3}
mkdir -p $O
L=paper_2107_01243_b200/_var/libsem_checked.so
for r in 1 2 3; do SEM_LIB=$L CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_loopback.py -m gpu -q -x > $O/blocking$r.log 2>&1; echo blocking$r=$? >> $O/rc.txt; done
SEM_LIB=$L timeout 1800 python -m pytest tests -m gpu -q > $O/checked_suite.log 2>&1; echo checked_suite=$? >> $O/rc.txt
cat $O/rc.txt
