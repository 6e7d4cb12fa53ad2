mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_hyena.py tests/test_gpu_backward.py -q --timeout 300 -p no:cacheprovider > gpurun_out/fir_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/fir_tests.log
timeout 300 python scripts/bench_kernels.py --which se > gpurun_out/bk_se.txt 2>&1; echo "bk rc=$?"; grep -E "featurizer|se_mixer_f32\"" gpurun_out/bk_se.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fir_stream -s 2 -c 1 -o gpurun_out/prof_feat python scripts/featprof.py > gpurun_out/ncu_feat.log 2>&1; echo "ncu feat rc=$?"
