cd $GRAFT_REPO_ROOT
MINBS="0" TESTS_K="wl or wide" NAME=wlsa4 bash scripts/gpu_r02_wlsa.sh
B="python bench.py --workload c5_679_zt --steps 2 --warmup 1 --phase-steps 2000 --no-cpu-baseline --no-e2e --no-per-config"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:walk_ -s 1 -c 1 -o gpurun_out/wlsa4.full_c5 -f $B > gpurun_out/wlsa4.ncu.log 2>&1
