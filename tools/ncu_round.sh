#!/bin/bash
# The round's ncu evidence (run on the GPU box from the repo root):
#  1. launch list of the default bench command (per-launch device times);
#  2. DRAM bytes per launch of the five hot-path kernels at the bench's per-GPU
#     sizes for N = 1, 2, 4, 8 (n_global = 2^33 strong scaling): one ncu pass
#     (3 metrics, no replay, so the 32-96 GiB buffers need no save/restore);
#  3. --set full of every hot-path kernel at 2^28 (tools/profile_ops.py).
# Summaries: tools/summarize_ncu.py (profiles/).
set -u
TAG=${1:-r2}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/${TAG}_launches_bench.log 2>&1
for L in 33 32 31 30; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:'ew_vec_kernel|reduce_kernel|scan_l2_kernel|scan_ring_kernel' -c 5 --csv --log-file gpurun_out/${TAG}_traffic_$L.csv \
      python bench.py --log2n-global $L --steps 3 --warmup 3 --no-cpu-baseline --no-extras \
      > gpurun_out/${TAG}_traffic_$L.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:'ew_vec_kernel|reduce_kernel|scan_l2_kernel|scan_ring_kernel' -c 5 \
    -o gpurun_out/${TAG}_full -f python tools/profile_ops.py 28 > gpurun_out/${TAG}_full.log 2>&1
echo done
