# A/B: stage z-march tile 32 x 4 at 4 CTAs per SM (MXB_ZTY=4, MXB_ZT_MINB=4), with 32 or 64 planes
set -x
P=gpurun_out/ztab
for V in zty4 zty4z64; do
  MXB_LIB=variants/$V/libmagnex_b200.so python -m pytest tests/test_zmarch.py -q > ${P}_tests_$V.txt 2>&1
done
for V in default zty4 zty4z64 default zty4 zty4z64 default zty4 zty4z64; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
