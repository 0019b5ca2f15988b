mkdir -p gpurun_out/ab
O=gpurun_out/ab/ab9.txt
run() { tag=$1; shift; echo "== $tag $*" >> $O; bash tools/quick_bench.sh "$@" >> $O 2>&1; }
run rmat rmat --kernel-times 20
run rmat-xna0 rmat --xload 0
run f32 rmat --dtype f32 --kernel-times 20
run f32-hot32-xna1 rmat --dtype f32 --hot-x 32 --xload 1
run f32-hot32-xna0 rmat --dtype f32 --hot-x 32 --xload 0
timeout 600 python tools/part_probe.py stencil csr 8 0,1,7 --sell 2,1 >> $O 2>&1
timeout 600 python tools/part_probe.py rmat csr 8 0,3,7 --sell 2 >> $O 2>&1
