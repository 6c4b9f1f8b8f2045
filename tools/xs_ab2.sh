# A/B: x-row fused stage (pair loads) against the unfused kernels (MXB_XFUSE=0)
set -x
P=gpurun_out/xsab2
timeout 900 python -m pytest tests/test_xstage.py tests/test_full_size.py -q -x > ${P}_tests_default.txt 2>&1
for r in 1 2; do
  for V in default unfused; do
    case $V in
      default) unset MXB_XFUSE ;;
      unfused) export MXB_XFUSE=0 ;;
    esac
    echo "$V $(timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
  done
done
