# A/B: r2c untangling twiddles by W^32 products between table anchors (MXB_XW_TWREC)
set -x
P=gpurun_out/trab
MXB_LIB=variants/twrec/libmagnex_b200.so python -m pytest tests/test_xwarp.py tests/test_bench_path_parity.py -q -k "not complex and not deviation" > ${P}_tests.txt 2>&1
for V in default twrec default twrec default twrec; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
