#!/bin/bash
# tools/evidence.sh: the committed measurement evidence of a round, on one B200 (run under gpurun):
#   default bench line, bench lines for every config / format / dtype, the ncu launch list of the
#   default bench, ncu --set full captures of the dominant kernels (+ traffic.json), the suite sweep,
#   the strong-scaling projection and the Fig. 6 imbalance study.  Output: gpurun_out/ev/
set -x
O=gpurun_out/ev; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
line() { timeout 900 python bench.py --steps ${STEPS:-500} --warmup 10 --e2e-steps 10 "$@" 2>/dev/null | tail -1 >> $O/bench_lines.jsonl; }
line --config stencil --kernel-times 20
line --config stencil --sell 1
line --config stencil --dtype f32 --sell 1
line --config stencil --format coo
line --config stencil --format csc
line --config stencil --dtype f32
line --config rmat --kernel-times 20
line --config rmat --format coo
line --config rmat --format csc
line --config rmat --format csc --col-layout 0
line --config rmat --format coo_col
line --config rmat --dtype f32
line --config rmat --layout owned
line --config rmatperm
line --config rmat --compact-x 2
line --config tallskinny
line --config tallskinny --col-layout 0
line --config tallskinny --dtype f32
line --config stencil --format csc --col-layout 0
line --config random1k --steps 5000
# launch list of the default bench (per-launch GPU time; cold-cache, serialised by ncu)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_rmat.csv \
  python bench.py --steps 10 --warmup 3 --e2e-steps 2 --no-cpu-baseline --xload 1 > /dev/null 2>&1
prof() {   # prof TAG KERNEL WORKLOAD_ARGS...
  tag=$1; k=$2; shift 2
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/prof_$tag -f \
    python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --xload 1 "$@" > $O/ncu_$tag.log 2>&1
  ncu -i $O/prof_$tag.ncu-rep --page details --csv > $O/${tag}_details.csv 2>&1
  ncu -i $O/prof_$tag.ncu-rep --page raw --csv > $O/${tag}_raw.csv 2>&1
  ncu -i $O/prof_$tag.ncu-rep --page source --csv --print-source sass > $O/${tag}_sass.csv 2>&1
}
prof rmat_rows rows_kernel
python tools/traffic_from_ncu.py $O/prof_rmat_rows.ncu-rep rmat_csr_f64_m16777216_n16777216_nnz263419028 rows_kernel > $O/traffic_rmat.txt 2>&1
prof stencil_rows rows_kernel --config stencil
python tools/traffic_from_ncu.py $O/prof_stencil_rows.ncu-rep stencil_csr_f64_m2048383_n2048383_nnz54439939 rows_kernel > $O/traffic_stencil.txt 2>&1
prof ts_csc rows_kernel --config tallskinny
python tools/traffic_from_ncu.py $O/prof_ts_csc.ncu-rep tallskinny_csc_f64_m50000000_n1000000_nnz500000000 rows_kernel > $O/traffic_ts.txt 2>&1
prof rmat_csc rows_kernel --config rmat --format csc
python tools/traffic_from_ncu.py $O/prof_rmat_csc.ncu-rep rmat_csc_f64_m16777216_n16777216_nnz263419028 rows_kernel > $O/traffic_rmat_csc.txt 2>&1
prof ts_bands csc_band_kernel --config tallskinny --col-layout 0
cp profiles/traffic.json $O/traffic.json
rm -f $O/*.ncu-rep
bash tools/suite_sweep.sh && mv gpurun_out/suite_sweep.jsonl $O/
timeout 2400 python tools/scaling_projection.py > $O/scaling_projection.jsonl 2> $O/scaling_projection.err
timeout 1200 python tools/imbalance_study.py > $O/imbalance_study.jsonl 2> $O/imbalance_study.err
