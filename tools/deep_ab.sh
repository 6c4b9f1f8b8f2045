# A/B: TMA z-march with deeper plane rings for the stages with <= 2 aux fields
# (variant deep: MXB_ZT_DEEP=1, state 3 / aux 2 planes ahead) against the default (2 / 1)
set -x
P=gpurun_out/deepab
timeout 900 python -m pytest tests/test_zmarch.py tests/test_full_size.py tests/test_xstage.py -q -x > ${P}_tests_default.txt 2>&1
MXB_LIB=variants/deep/libmagnex_b200.so timeout 900 python -m pytest tests/test_zmarch.py tests/test_full_size.py tests/test_xstage.py -q -x > ${P}_tests_deep.txt 2>&1
for r in 1 2 3; do
  for V in default deep; do
    case $V in
      default) unset MXB_LIB ;;
      *) export MXB_LIB=variants/$V/libmagnex_b200.so ;;
    esac
    echo "$V $(timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
  done
done
