# round-2 final measurement set (one box): GPU suite, smoke, bench lines c1-c5,
# reference arm, bench launch list, ncu full page of the c2 kernel
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/final/pytest_gpu_full.log 2>&1; echo "rc=$?" >> gpurun_out/final/pytest_gpu_full.log
for c in c2 c1 c3 c4 c5; do
  timeout 600 python bench.py --config $c > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
done
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_reference_c2.json 2> gpurun_out/final/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/bench_launches.csv python bench.py --steps 5 --warmup 3 --no-ncu --no-bounds --paper-rule-s 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_sym -s 2 -c 1 -o gpurun_out/final/c2_full python tools/profile_one.py --config c2 > gpurun_out/final/c2_full.log 2>&1
python tools/prepare_time.py > gpurun_out/final/prepare_time.jsonl 2> gpurun_out/final/prepare_time.err
for c in c2 c3 c4 c5; do python tools/profile_oneshot.py $c 20; done > gpurun_out/final/one_shot.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/oneshot_launches_c2.csv python tools/profile_oneshot.py c2 1 > /dev/null 2>&1
echo done
