#!/bin/bash
# tools/aux_benches.sh: the NEXT-f benches of the current build (CG, SpMM, host-resident) -> gpurun_out/aux/
O=gpurun_out/aux; mkdir -p $O
for f in csr coo csc; do timeout 600 python tools/cg_bench.py --format $f >> $O/cg_bench.jsonl 2>> $O/cg.err; done
timeout 600 python tools/cg_bench.py --format csr --graph 0 >> $O/cg_bench.jsonl 2>> $O/cg.err
timeout 600 python tools/spmm_bench.py --config stencil > $O/spmm_bench.jsonl 2>> $O/spmm.err
timeout 900 python tools/spmm_bench.py --config rmat >> $O/spmm_bench.jsonl 2>> $O/spmm.err
timeout 900 python tools/host_resident_bench.py > $O/host_resident.jsonl 2> $O/host_resident.err
