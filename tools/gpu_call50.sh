mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "cg" > gpurun_out/pytest_cg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cg.log
rm -f gpurun_out/cg_graph.jsonl
for N in 127 48 24 12; do for g in 1 0; do
  MSREP_CG_GRAPH=$g timeout 300 python tools/cg_bench.py --N $N --iters 400 >> gpurun_out/cg_graph.jsonl 2>&1
done; done
for f in coo csc; do for g in 1 0; do MSREP_CG_GRAPH=$g timeout 300 python tools/cg_bench.py --format $f --iters 200 >> gpurun_out/cg_graph.jsonl 2>&1; done; done
