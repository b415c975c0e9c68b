mkdir -p gpurun_out/s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/s3/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/s3/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s3/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/s3/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/s3/bench_default.json 2> gpurun_out/s3/bench_default.err; echo "rc=$?" >> gpurun_out/s3/bench_default.err
echo done
