# usage: bash tools/gpu_variants_modes.sh "-DX=1" ...  rebuild per flag set on the box; force /
# detect / step device times for configs[1] fp64, fp32 mode and configs[2] (tools/modes_kernel_ms.py)
for v in "$@"; do
  touch paper_1503_03553_b200/csrc/*.cu
  make -C paper_1503_03553_b200 -j8 EXTRA="$v" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "[$v] $(timeout 300 python tools/modes_kernel_ms.py ${MODES:-} 2>&1 | tail -1)"
done
