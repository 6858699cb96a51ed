O=gpurun_out/${CD_TAG:-chkdbg}
mkdir -p $O
L=paper_2107_01243_b200/_var/libsem_checked.so
SEM_LIB=$L timeout 900 python -m pytest tests/test_gpu_schwarz.py -m gpu -q -x > $O/schwarz.log 2>&1; echo schwarz=$? >> $O/rc.txt
SEM_LIB=$L timeout 900 python -m pytest tests/test_loopback.py -m gpu -q -x -k "P2" > $O/loop_p2.log 2>&1; echo loop2=$? >> $O/rc.txt
SEM_LIB=$L CUDA_LAUNCH_BLOCKING=1 timeout 900 python -m pytest tests/test_loopback.py -m gpu -q -x -k "P2" > $O/loop_p2_blocking.log 2>&1; echo loop2b=$? >> $O/rc.txt
timeout 900 python -m pytest tests/test_loopback.py -m gpu -q -x > $O/loop_default.log 2>&1; echo loopdef=$? >> $O/rc.txt
cat $O/rc.txt
