# time variant builds: tools/gpu/variants.sh "<iter args>" libA.so libB.so ...
args="$1"; shift
python tools/gpu/iter.py $args
for v in "$@"; do echo "== $v"; HAPT_LIB=paper_2509_24859_b200/$v python tools/gpu/iter.py --no-parity $args; done
