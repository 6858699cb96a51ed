O=gpurun_out/${CD_TAG:-chkdbg2}
mkdir -p $O
L=paper_2107_01243_b200/_var/libsem_checked.so
CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_loopback.py -m gpu -q -x -k "P2" > $O/reg_blocking.log 2>&1; echo reg_blocking=$? >> $O/rc.txt
SEM_LIB=paper_2107_01243_b200/_var/libsem_chknc.so CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_loopback.py -m gpu -q -x -k "P2" > $O/chknc_blocking.log 2>&1; echo chknc_blocking=$? >> $O/rc.txt
SEM_LIB=$L CUDA_LAUNCH_BLOCKING=1 timeout 900 cuda-gdb -batch -ex "set pagination off" -ex run -ex "thread apply all bt 25" --args python -m pytest tests/test_loopback.py -m gpu -q -x -k P2 > $O/gdb.log 2>&1; echo gdb=$? >> $O/rc.txt
cat $O/rc.txt
