#!/bin/bash
# A/B sweep of NCCL channel / protocol settings for the gradient all-reduce at
# N GPUs (C2 bench, one line per setting). Usage: scripts/nccl_sweep.sh N OUTDIR
# [tag:VAR=value ...] (no settings: the NCCL sweep below)
N=${1:-2}; OUT=${2:-gpurun_out}; shift 2 2>/dev/null
run() {
  local tag=$1; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" \
    --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus "$N" --steps 300 --warmup 10 \
    --no-cpu-baseline > "$OUT/sweep_n${N}_${tag}.json" 2> "$OUT/sweep_n${N}_${tag}.err"
  python - "$OUT/sweep_n${N}_${tag}.json" "$tag" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:>12} value {d['value']:.0f} ms/step {d['ms_per_step']*1e3:.1f}us e2e {d['e2e']['value']:.0f} adam {d['phases_ms_graph_critical_path']['adam']*1e3:.1f}us")
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
}
if [ $# -gt 0 ]; then
  for kv in "$@"; do run "${kv%%:*}" "${kv#*:}"; done
  exit 0
fi
run default X=1
run minch16 NCCL_MIN_NCHANNELS=16
run minch32 NCCL_MIN_NCHANNELS=32
run maxch4 NCCL_MAX_NCHANNELS=4
run ll128 NCCL_PROTO=LL128
run ll NCCL_PROTO=LL
run nonvls NCCL_NVLS_ENABLE=0
run peer TGNN_ALLREDUCE=peer
run default2 X=1
