# A/B: x c2r prefetch of the spectrum slice pfd CTAs ahead by per-thread L2 line
# prefetches (variant c2rl, MXB_XW_PFD_C2R = 148 / 296) against no c2r prefetch
set -x
P=gpurun_out/c2rlab
MXB_LIB=variants/c2rl/libmagnex_b200.so MXB_XW_PFD_C2R=148 timeout 900 python -m pytest tests/test_pipe.py tests/test_bench_path_parity.py tests/test_full_size.py -q -x > ${P}_tests_c2rl.txt 2>&1
for r in 1 2 3; do
  for V in default c148 c296; do
    case $V in
      default) unset MXB_LIB; unset MXB_XW_PFD_C2R ;;
      c*) export MXB_LIB=variants/c2rl/libmagnex_b200.so; export MXB_XW_PFD_C2R=${V#c} ;;
    esac
    echo "$V $(timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
  done
done
