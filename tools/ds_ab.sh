# A/B: C-unit discard after the inverse FFT (MXB_PIPE_DISCARD_LATE) and release reductions for the
# completion signals (MXB_PIPE_SIGNAL_REL) in the plane pipeline
set -x
P=gpurun_out/dsab
for V in dlate srel both; do
  MXB_LIB=variants/$V/libmagnex_b200.so python -m pytest tests/test_pipe.py tests/test_bench_path_parity.py -q -k "warp or l1024" > ${P}_tests_$V.txt 2>&1
done
for V in default dlate srel both default dlate srel both default dlate srel both; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  echo "$V $(python bench.py --steps 10 --warmup 3 --repeats 3 --no-e2e --no-cpu --no-dev --no-ref-mode 2>>${P}_bench.err)" >> ${P}_bench_all.txt
done
unset MXB_LIB
for V in default dlate srel both; do
  if [ $V = default ]; then unset MXB_LIB; else export MXB_LIB=variants/$V/libmagnex_b200.so; fi
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"k_yz_pipe_w" -c 2 --csv --log-file ${P}_ncu_$V.csv python tools/profile_step.py --n 512 --steps 1 > ${P}_ncu_$V.log 2>&1
done
