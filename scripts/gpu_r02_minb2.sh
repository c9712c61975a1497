cd $GRAFT_REPO_ROOT
: > gpurun_out/minb2.log
for rep in 1 2; do for mb in ${MBS:-0 16 24}; do
  out=$(FG_WL_MINB=$mb timeout 300 python bench.py --workload c4_555_zt --steps 3 --warmup 3 --phase-steps 2000 --no-cpu-baseline --no-e2e --no-per-config 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e6,1), 'M', round(r['kernel_ms_per_launch'],3), 'ms')")
  echo "rep $rep minb $mb $out" >> gpurun_out/minb2.log
done; done
