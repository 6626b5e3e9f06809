# ncu evidence for the shipped DP kernel generation: launch list, per-launch
# traffic of every relax launch, one --set full capture of a mid-sweep
# dp_relax_compact launch (D1 pool).  -> gpurun_out/$1_*
tag=${1:-prof}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv python tools/profile_dp.py --config D1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__t_bytes.sum,smsp__inst_executed.sum --clock-control none -k regex:dp_relax --csv --log-file gpurun_out/${tag}_traffic.csv python tools/profile_dp.py --config D1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:dp_relax_compact --launch-skip 30 --launch-count 1 -o gpurun_out/${tag}_full python tools/profile_dp.py --config D1 > gpurun_out/${tag}_full.log 2>&1
ls -la gpurun_out/${tag}_*
