# A/B: four twiddle chains in fft1024 (MXB_FFT_TW4) and two chains in fft512x2
# (MXB_FFT512_TW2: x passes at nx = 512 and the L = 512 pipeline)
set -x
P=gpurun_out/tw4ab
MXB_LIB=variants/tw4/libmagnex_b200.so python -m pytest tests/test_pipe.py tests/test_bench_path_parity.py -q -k "warp or l1024" > ${P}_tests_tw4.txt 2>&1
MXB_LIB=variants/f512/libmagnex_b200.so python -m pytest tests/test_pipe.py tests/test_xwarp.py tests/test_bench_path_parity.py -q -k "warp or l1024 or x_passes or l512" > ${P}_tests_f512.txt 2>&1
for V in default tw4 f512 default tw4 f512 default tw4 f512; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
for V in default f512 default f512; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --size 256 --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench256.txt
done
