mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest_gpu8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab/pytest_gpu8.log
(cd tools/variants/dbgtime && timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | grep -E 'msrep phase4|partition_ms' | cut -c1-300) > gpurun_out/ab/phase4.txt 2>&1
(cd tools/variants/dbgtime && timeout 600 python bench.py --config tallskinny --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | grep -E 'msrep phase4') >> gpurun_out/ab/phase4.txt 2>&1
