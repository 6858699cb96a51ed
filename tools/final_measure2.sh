# End-of-round single-GPU measurement (run under gpurun from the repo root).
O=gpurun_out/fin
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests=$? >> $O/rc.txt
timeout 600 python bench.py > $O/bench1.json 2> $O/bench1.err; echo bench1=$? >> $O/rc.txt
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$? >> $O/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo launches=$? >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ax_kernel|gs_update|cg_p|gs_local|cg_update" -c 10 -o $O/prof_pcg python tools/prof.py C2 > $O/ncu_full.log 2>&1; echo full=$? >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fdm8|combine|mdot|maxpy" -c 12 -o $O/prof_schwarz python tools/prof_schwarz.py > $O/ncu_schwarz.log 2>&1; echo fullschw=$? >> $O/rc.txt
timeout 600 python tools/measure.py schwarz C2,C3,C4 > $O/schwarz.jsonl 2> $O/schwarz.err; echo schwarz=$? >> $O/rc.txt
timeout 1200 python tools/measure.py single > $O/measure_single.jsonl 2> $O/measure_single.err; echo single=$? >> $O/rc.txt
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem,power.limit --format=csv > $O/smi.txt 2>&1
