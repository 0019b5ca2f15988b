mkdir -p gpurun_out/ab
O=gpurun_out/ab/ab14.txt
run() { tag=$1; shift; echo "== $tag $*" >> $O; bash tools/quick_bench.sh "$@" >> $O 2>&1; }
for rep in 1 2; do
for c in 1 2; do
run "rmat-c$c" rmat --compact-x $c
run "rmatf32-c$c" rmat --dtype f32 --compact-x $c
run "rmatperm-c$c" rmatperm --compact-x $c
run "pl-c$c" suite-powerlaw-100M --compact-x $c
run "rmatcsc-c$c" rmat --format csc --compact-x $c
done
done
