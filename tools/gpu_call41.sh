mkdir -p gpurun_out
rm -f gpurun_out/fsell.txt
for c in "rmat" "suite-powerlaw-100M" "suite-shortwide-100M"; do
  bash tools/quick_bench.sh $c >> gpurun_out/fsell.txt 2>&1
  MSREP_LIB_VARIANT=tools/libmsrep_fsell.so bash tools/quick_bench.sh $c | sed "s/^/fsell /" >> gpurun_out/fsell.txt 2>&1
done
timeout 600 python tools/dbg_part.py rmat 4 3 > gpurun_out/dbg_part.txt 2>&1
timeout 1500 python tools/scaling_projection.py --configs rmat:csr > gpurun_out/scaling_projection_rmat.jsonl 2> gpurun_out/scaling_projection.err
