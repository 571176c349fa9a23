# One GPU call: bench (full contract incl. cpu_baseline), reference arm, ncu launch list of the
# bench command, ncu --set full of the two hot kernels. Outputs in gpurun_out/ ($1 = round tag).
tag=${1:-r01}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_$tag.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-north-star > gpurun_out/launch_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_force_reduce|k_detect|k_integrate_hash|k_reorder" \
    -s 12 -c 4 -o gpurun_out/prof_$tag python tools/prof_driver.py --warmup 3 --steps 2 > gpurun_out/prof_$tag.log 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host_$tag.txt
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv >> gpurun_out/host_$tag.txt
tail -c 600 gpurun_out/bench_$tag.json; tail -c 300 gpurun_out/bench_ref_$tag.json; tail -2 gpurun_out/prof_$tag.log
