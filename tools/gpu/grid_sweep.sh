# dp_relax_compact grid cap sweep of a variant build: tools/gpu/grid_sweep.sh lib.so "g1 g2 ..." "<iter args>"
lib=$1; grids=$2; args=$3
for g in $grids; do echo "== $lib grid $g"; HAPT_RELAX_GRID=$g HAPT_LIB=paper_2509_24859_b200/$lib python tools/gpu/iter.py --no-parity $args 2>&1 | grep -v Warn; HAPT_RELAX_GRID=$g HAPT_LIB=paper_2509_24859_b200/$lib python tools/gpu/subset.py D1 2,4,8 2>&1 | grep -v Warn | sed 's/\[prof.*//'; done
