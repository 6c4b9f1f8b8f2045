# ncu evidence for the long-y (film) path: launch list of one demag-only probe,
# then a full capture of one launch of each long-y kernel (run after the probe
# itself exited 0 without ncu)
set -x
timeout 300 python tools/pipe_probe.py 2048 2048 64 > gpurun_out/film_probe.txt 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2m_film_launches.csv \
    python tools/pipe_probe.py 2048 2048 64 > gpurun_out/ncu_f1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_yrow|k_fused_fast|k_rm_to_pm" -c 4 \
    -o gpurun_out/r2m_film python tools/pipe_probe.py 2048 2048 64 > gpurun_out/ncu_f2.log 2>&1
