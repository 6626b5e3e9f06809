# ncu launch list of one D1 full-pool sweep -> gpurun_out/$1.csv, plus per-kernel summary
tag=${1:-launches}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag.csv python tools/profile_dp.py --config ${2:-D1} > /dev/null 2>&1
python tools/kernel_share.py gpurun_out/$tag.csv
