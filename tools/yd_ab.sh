# A/B: TMA z-march stage without the step-start-state box in the first stage (default,
# MXB_ZT_YDEDUP=1) against the build that loads it (nodedup)
set -x
P=gpurun_out/ydab
timeout 900 python -m pytest tests/test_zmarch.py tests/test_full_size.py tests/test_gpu_parity.py tests/test_xstage.py -q -x > ${P}_tests_default.txt 2>&1
for r in 1 2 3; do
  for V in default nodedup; do
    case $V in
      default) unset MXB_LIB ;;
      *) export MXB_LIB=variants/$V/libmagnex_b200.so ;;
    esac
    echo "$V $(timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
  done
done
