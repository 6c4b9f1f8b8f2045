# A/B: x passes -- L2 prefetch of the input pfd CTAs ahead (MXB_XW_PFD, run time) and
# the plane-major r2c storing its outputs from registers (variant r2cd)
set -x
P=gpurun_out/xwab
MXB_LIB=variants/r2cd/libmagnex_b200.so timeout 900 python -m pytest tests/test_pipe.py tests/test_bench_path_parity.py tests/test_full_size.py -q -x > ${P}_tests_r2cd.txt 2>&1
MXB_XW_PFD=592 timeout 900 python -m pytest tests/test_pipe.py tests/test_full_size.py -q -x > ${P}_tests_pfd.txt 2>&1
for r in 1 2; do
  for V in d0 d296 d592 d1184 r2cd0 r2cd592; do
    case $V in
      d*) unset MXB_LIB; export MXB_XW_PFD=${V#d} ;;
      r2cd*) export MXB_LIB=variants/r2cd/libmagnex_b200.so; export MXB_XW_PFD=${V#r2cd} ;;
    esac
    echo "$V $(timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
  done
done
