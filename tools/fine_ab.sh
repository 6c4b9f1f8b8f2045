# A/B: r2c prefetch distance around the default (MXB_XW_PFD, run time) and 128 z planes
# per stage CTA (variant zc128: MXB_ZC=128)
set -x
P=gpurun_out/fineab
MXB_LIB=variants/zc128/libmagnex_b200.so timeout 900 python -m pytest tests/test_zmarch.py tests/test_full_size.py -q -x > ${P}_tests_zc128.txt 2>&1
for r in 1 2 3; do
  for V in x148 x74 x110 x200 zc128; do
    case $V in
      x*) unset MXB_LIB; export MXB_XW_PFD=${V#x} ;;
      *) export MXB_LIB=variants/$V/libmagnex_b200.so; unset MXB_XW_PFD ;;
    esac
    echo "$V $(timeout 300 python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
  done
done
