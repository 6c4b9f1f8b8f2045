# A/B: x-row fused stage variants (L2 prefetch off: pf0; software-pipelined loads: swp)
# against the default build and the unfused kernels (MXB_XFUSE=0)
set -x
P=gpurun_out/xsab
for V in pf0 swp; do
  MXB_LIB=variants/$V/libmagnex_b200.so timeout 600 python -m pytest tests/test_xstage.py -q -x > ${P}_tests_$V.txt 2>&1
done
timeout 900 python -m pytest tests/test_xstage.py tests/test_full_size.py -q -x > ${P}_tests_default.txt 2>&1
for r in 1 2; do
  for V in default unfused pf0 swp; do
    case $V in
      default) unset MXB_LIB; unset MXB_XFUSE ;;
      unfused) unset MXB_LIB; export MXB_XFUSE=0 ;;
      *) export MXB_LIB=variants/$V/libmagnex_b200.so; unset MXB_XFUSE ;;
    esac
    echo "$V $(timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
  done
done
