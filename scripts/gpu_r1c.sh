cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -k "addmul or product or trunc" -x -q > $O/r1c_pytest.log 2>&1; echo "pytest $?"; tail -2 $O/r1c_pytest.log
HM_DUMP_EVAL=$O/r1c_evaldump.txt timeout 600 python bench.py --no-factor --no-cpu-baseline --steps 1 --warmup 3 > $O/r1c_bench_split.json 2>&1; echo "bench $?"
HM_EVAL_SPLIT=0 timeout 600 python bench.py --no-factor --no-cpu-baseline --steps 2 --warmup 3 > $O/r1c_bench_nosplit.json 2>&1
timeout 600 python bench.py --no-factor --no-cpu-baseline --steps 2 --warmup 3 > $O/r1c_bench_split2.json 2>&1
timeout 600 python scripts/ncu_step.py save /tmp/cfg4.npz > /dev/null 2>&1
HM_NCU_NOWARM=1 timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $O/r1c_launches.csv python scripts/ncu_step.py load /tmp/cfg4.npz > $O/r1c_ncu_list.log 2>&1
echo "ncu $?"
