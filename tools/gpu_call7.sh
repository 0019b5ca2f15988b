mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "csc" > gpurun_out/pytest_csc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_csc.log
rm -f gpurun_out/qb_var.txt
for c in "tallskinny" "tallskinny --dtype f32"; do bash tools/quick_bench.sh $c >> gpurun_out/qb_var.txt 2>&1; done
bash tools/gpu_prof.sh ts_band4 csc_band_kernel --config tallskinny
