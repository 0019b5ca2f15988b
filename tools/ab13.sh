mkdir -p gpurun_out/ab
O=gpurun_out/ab/ab13.txt
run() { tag=$1; shift; echo "== $tag $*" >> $O; bash tools/quick_bench.sh "$@" >> $O 2>&1; }
for rep in 1 2; do
run deg rmat --compact-x 2
run inter rmat --compact-x 3
run col rmat --compact-x 1
run pl-deg suite-powerlaw-100M --compact-x 2
run pl-inter suite-powerlaw-100M --compact-x 3
done
O2=gpurun_out/ab13; mkdir -p $O2
timeout 900 ncu --set full --clock-control none -k regex:rows_kernel -s 3 -c 1 -o $O2/prof_inter -f \
    python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --compact-x 3 > $O2/ncu.log 2>&1
ncu -i $O2/prof_inter.ncu-rep --page raw --csv > $O2/inter_raw.csv 2>&1
ncu -i $O2/prof_inter.ncu-rep --page details --csv > $O2/inter_details.csv 2>&1
rm -f $O2/prof_inter.ncu-rep
