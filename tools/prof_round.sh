set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_all.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
python bench.py > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
python bench.py --steps 2 --warmup 3 --repeats 1 --no-e2e --no-cpu > gpurun_out/r2j_b2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2j_launches.csv python bench.py --steps 2 --warmup 3 --repeats 1 --no-e2e --no-cpu > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_r2c_w|k_yz_pipe_w|k_c2r_w|k_stage_zt" -c 7 -o gpurun_out/r2j_prof512 python tools/profile_step.py --n 512 --steps 1 > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out/
