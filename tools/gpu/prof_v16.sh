set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/profile_dp.py --config D1 --time 20 > gpurun_out/r2_v16_time.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__t_bytes.sum,smsp__inst_executed.sum --clock-control none -k regex:dp_relax --csv --log-file gpurun_out/r2_v16_relax_traffic.csv python tools/profile_dp.py --config D1 > gpurun_out/r2_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:dp_relax_compact --launch-skip 30 --launch-count 1 -o gpurun_out/r2_v16_relax_full python tools/profile_dp.py --config D1 > gpurun_out/r2_ncu2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_v16_launches.csv python tools/profile_dp.py --config D1 > gpurun_out/r2_ncu3.log 2>&1
ls -la gpurun_out
