set -u
mkdir -p gpurun_out
timeout 900 python tools/sweep.py --out gpurun_out/sweep_r2b.json > gpurun_out/sweep_r2b.log 2>&1; echo "sweep rc=$?" >> gpurun_out/job.log
for t in memcheck racecheck synccheck; do
  echo "== $t" >> gpurun_out/sanitizer_r2b.log
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_drive.py 2>&1 | tail -4 >> gpurun_out/sanitizer_r2b.log
done
echo "sanitizer done" >> gpurun_out/job.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'scan_ring_kernel' -c 2 -o gpurun_out/ring26_full -f python tools/profile_ops.py 26 scan > gpurun_out/ring26_full.log 2>&1; echo "ncu26 rc=$?" >> gpurun_out/job.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'scan_ring_kernel' -c 2 -o gpurun_out/ring25_64_full -f python tools/profile_ops.py 25 scan64 > gpurun_out/ring25_64_full.log 2>&1; echo "ncu25-64 rc=$?" >> gpurun_out/job.log
