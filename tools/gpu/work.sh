for v in "$@"; do echo "== $v"; HAPT_LIB=paper_2509_24859_b200/$v python tools/work_counts.py D1 C 2>&1 | grep -v source; done
