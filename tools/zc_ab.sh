# A/B: z planes per CTA of the TMA z-march stage kernel (MXB_ZC, default 16)
set -x
P=gpurun_out/zcab
for V in zc32 zc64 zc8; do
  MXB_LIB=variants/$V/libmagnex_b200.so python -m pytest tests/test_zmarch.py -q > ${P}_tests_$V.txt 2>&1
done
for V in default zc32 zc64 zc8 default zc32 zc64 zc8 default zc32 zc64 zc8; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
