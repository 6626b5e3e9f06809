# tools/gpu/subset_envs.sh <config> <worlds> "ENV=V ..." ...
cfg=$1; w=$2; shift 2
python tools/gpu/subset.py $cfg $w
for v in "$@"; do echo "== $v"; env $v python tools/gpu/subset.py $cfg $w; done
