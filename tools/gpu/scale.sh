# strong-scaling lines of bench.py on every GPU count up to the box's: tools/gpu/scale.sh <tag> <configs...>
tag=$1; shift
ngpu=$(nvidia-smi -L | wc -l)
for cfg in "$@"; do
  for n in 1 2 4 8; do
    [ $n -gt $ngpu ] && break
    if [ $n -eq 1 ]; then
      python bench.py --config $cfg --steps 20 --warmup 5 --no-extras > gpurun_out/${tag}_${cfg}_n1.json 2> gpurun_out/${tag}_${cfg}_n1.err
    else
      python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
        bench.py --gpus $n --config $cfg --steps 20 --warmup 5 --no-extras > gpurun_out/${tag}_${cfg}_n$n.json 2> gpurun_out/${tag}_${cfg}_n$n.err
    fi
    python - "$cfg" "$n" "gpurun_out/${tag}_${cfg}_n$n.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    print(sys.argv[1], "N=" + sys.argv[2], round(d["value"]), "cand/s", round(d["ms_per_step"], 3), "ms",
          "e2e", round(d["e2e"]["value"]), "search", round(d["search_time_s"] * 1e3, 2), "ms", d["clocks"])
except Exception as e:
    print(sys.argv[1], sys.argv[2], "failed", e)
PY
  done
done
