mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/cooq.txt
for c in "stencil --format coo" "suite-banded-100M --format coo" "suite-blockdiag-100M --format coo" "rmat --format coo" "suite-powerlaw-100M --format coo" "suite-shortwide-100M --format coo" "stencil --format coo --dtype f32"; do
  bash tools/quick_bench.sh $c >> gpurun_out/cooq.txt 2>&1
done
timeout 600 python tools/dbg_part.py rmat 4 3 > gpurun_out/dbg_part.txt 2>&1
timeout 600 python tools/dbg_part.py rmat 4 2 >> gpurun_out/dbg_part.txt 2>&1
