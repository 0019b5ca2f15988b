mkdir -p gpurun_out/ab
O=gpurun_out/ab/abhc.txt; : > $O
for rep in 1 2; do
for v in . tools/variants/hc32; do
  for c in "rmat" "tallskinny"; do
    echo "== $v $c" >> $O
    (cd $v && timeout 600 python bench.py --config $c --steps 50 --warmup 5 --e2e-steps 20 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:30], 'e2e_ms', round(d['e2e']['ms_per_step'],3))") >> $O 2>&1
  done
done
done
