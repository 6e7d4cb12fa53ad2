mkdir -p gpurun_out
timeout 300 python scripts/bench_kernels.py --which li > gpurun_out/bk_li.txt 2>&1; echo "bk li rc=$?"; cat gpurun_out/bk_li.txt
timeout 300 python scripts/bench_kernels.py --which se > gpurun_out/bk_se.txt 2>&1; echo "bk se rc=$?"; cat gpurun_out/bk_se.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:two_stage_kernel -s 5 -c 1 -o gpurun_out/prof_li python scripts/bench_kernels.py --which li > gpurun_out/ncu_li.log 2>&1; echo "ncu li rc=$?"; tail -3 gpurun_out/ncu_li.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:se_mixer_kernel -s 5 -c 1 -o gpurun_out/prof_se python scripts/bench_kernels.py --which se > gpurun_out/ncu_se.log 2>&1; echo "ncu se rc=$?"; tail -3 gpurun_out/ncu_se.log
