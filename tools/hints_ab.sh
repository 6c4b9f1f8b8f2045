# A/B of per-access L2 eviction hints in k_yz_pipe_w (MXB_PIPE_HINTS variants,
# tools/build_variant.py h1 / h2 / h1k yz_pipe.cu -DMXB_PIPE_HINTS=...).
set -x
P=gpurun_out/hints3
for V in kph1k kph2 nohint; do
  MXB_LIB=variants/$V/libmagnex_b200.so python -m pytest tests/test_pipe.py -q -k "warp" > ${P}_tests_$V.txt 2>&1
done
for V in default kph1k kph2 nohint default kph1k kph2 nohint; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 5 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
unset MXB_LIB
for V in default kph1k kph2 nohint; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none \
      -k regex:"k_yz_pipe_w" -c 2 --csv --log-file ${P}_ncu_$V.csv python tools/profile_step.py --n 512 --steps 1 > ${P}_ncu_$V.log 2>&1
done
# L = 512 pair kernel (256^3 grid)
for V in default kp512 default kp512; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --size 256 --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench256.txt
done
unset MXB_LIB
MXB_LIB=variants/kp512/libmagnex_b200.so python -m pytest tests/test_pipe.py -q -k "l512" > ${P}_tests_kp512.txt 2>&1
