#!/bin/bash
# bench.py plain vs under torchrun (1 rank, NCCL pool sync every phase), alternated on one box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/trab.log; : > $O
for rep in 1 2 3; do
  v=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-per-config --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,4), round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_per_launch'],3))")
  echo "rep $rep plain    $v" >> $O
  v=$(timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2953$rep bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline --no-per-config --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,4), round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_per_launch'],3))")
  echo "rep $rep torchrun $v" >> $O
done
