# ncu --set full of one mid-sweep dp_relax_compact launch (D1 pool) -> gpurun_out/$1.ncu-rep
tag=${1:-relax_full}
ncu --set full --import-source on --clock-control none -k regex:dp_relax_compact --launch-skip ${2:-30} --launch-count 1 -o gpurun_out/$tag python tools/profile_dp.py --config ${3:-D1} > gpurun_out/$tag.log 2>&1
tail -2 gpurun_out/$tag.log
