# needs: python tools/build_variant.py xw0 x_warp.cu -DMXB_XW_EXIT_READ=0
set -x
python -m pytest tests/test_xwarp.py tests/test_pipe.py -x -q > gpurun_out/xe_tests.txt 2>&1
for V in xw0 default xw0 default xw0 default; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 5 --warmup 3 --repeats 3 --no-e2e --no-cpu 2>>gpurun_out/xe_bench.err)" >> gpurun_out/xe_bench_all.txt
done
