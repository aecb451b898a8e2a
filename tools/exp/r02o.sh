mkdir -p gpurun_out
[ -z "$SKIP_TESTS" ] && timeout 900 python -m pytest tests/test_gpu_apps.py -k binomial -x -q -p no:cacheprovider > gpurun_out/${TAG:-r02o}_tests.txt 2>&1; echo rc=$? >> gpurun_out/${TAG:-r02o}_tests.txt
[ -z "$SKIP_TESTS" ] && timeout 600 python -m pytest "tests/test_gpu_fullshape.py::test_c2_binomial_headline_shape" -x -q -p no:cacheprovider >> gpurun_out/${TAG:-r02o}_tests.txt 2>&1; echo rc=$? >> gpurun_out/${TAG:-r02o}_tests.txt
for v in ${VARIANTS:-default seg8 seg0}; do
  if [ $v = default ]; then L=; else L=tools/variants/$v/libhpac_b200.so; fi
  env ${L:+HPAC_LIB=$L} timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --sub-configs off > gpurun_out/${TAG:-r02o}_bench_$v.json 2> gpurun_out/${TAG:-r02o}_bench_$v.err
done
