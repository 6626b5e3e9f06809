# time env-var variants: tools/gpu/envs.sh "<iter args>" "ENV=V ..." "ENV=V ..." ...
args="$1"; shift
python tools/gpu/iter.py $args
for v in "$@"; do echo "== $v"; env $v python tools/gpu/iter.py --no-parity $args; done
