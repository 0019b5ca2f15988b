O=gpurun_out/ab12; mkdir -p $O
prof() {   # prof TAG KERNEL ARGS...
  tag=$1; k=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/prof_$tag -f \
    python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline "$@" > $O/ncu_$tag.log 2>&1
  ncu -i $O/prof_$tag.ncu-rep --page details --csv > $O/${tag}_details.csv 2>&1
  ncu -i $O/prof_$tag.ncu-rep --page raw --csv > $O/${tag}_raw.csv 2>&1
  ncu -i $O/prof_$tag.ncu-rep --page source --csv --print-source sass > $O/${tag}_sass.csv 2>&1
  rm -f $O/prof_$tag.ncu-rep
}
prof f32hot rows_kernel --dtype f32 --hot-x 32 --xload 1
prof f32cold rows_kernel --dtype f32 --xload 1
