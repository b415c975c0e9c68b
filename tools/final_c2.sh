# c2 bench line, launch list and ncu full page after the launch rule change
mkdir -p gpurun_out/final2
timeout 600 python bench.py --config c2 > gpurun_out/final2/bench_c2.json 2> gpurun_out/final2/bench_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final2/bench_launches.csv python bench.py --steps 5 --warmup 3 --no-ncu --no-bounds --paper-rule-s 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_sym -s 2 -c 1 -o gpurun_out/final2/c2_full python tools/profile_one.py --config c2 > gpurun_out/final2/c2_full.log 2>&1
