# ncu --set full of the step kernels of the bench workload (tag = $1, kernel regex = $2)
tag=${1:-x}; rx=${2:-"k_force_reduce|k_detect"}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s ${SKIP:-10} -c ${COUNT:-2} \
    -o gpurun_out/prof_$tag python tools/prof_driver.py --warmup 5 --steps 2 ${PROF_ARGS:-} > gpurun_out/prof_$tag.log 2>&1
tail -1 gpurun_out/prof_$tag.log
