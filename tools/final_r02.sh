# Round-2 single-GPU evidence run (under gpurun from the repo root):
# GPU suite, smoke, bench (+ reference arm), ncu launch list of the bench
# command, ncu --set full of the PCG kernels, Schwarz kernels, then the
# summary into profiles/.
O=gpurun_out/${1:-fin2}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem,power.limit --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests=$? >> $O/rc.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/rc.txt
timeout 900 python bench.py > $O/bench1.json 2> $O/bench1.err; echo bench1=$? >> $O/rc.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$? >> $O/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3 > $O/ncu_launch.log 2>&1; echo launches=$? >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ax_kernel|gs_local|cg_update|cg_p" -c 24 -o $O/prof_pcg python tools/prof.py C2 > $O/ncu_full.log 2>&1; echo full=$? >> $O/rc.txt
cat $O/rc.txt
timeout 1200 python tools/measure.py ops C3,C4 > $O/ops.jsonl 2> $O/ops.err; echo ops=$? >> $O/rc.txt
timeout 1200 python tools/measure.py schwarz C2,C3,C4 > $O/schwarz.jsonl 2> $O/schwarz.err; echo schwarz=$? >> $O/rc.txt
timeout 900 python tools/measure.py helm C3 > $O/helm.jsonl 2> $O/helm.err; echo helm=$? >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ax_kernel<8, 2, 0, 1>|gs_local|cg_update" -c 3 -o $O/prof_pf python tools/prof.py C2 > $O/ncu_pf.log 2>&1; echo full_pf=$? >> $O/rc.txt
cat $O/rc.txt
