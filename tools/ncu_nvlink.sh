#!/bin/bash
# NVLink bytes per layer stage on a multi-GPU box (one GPU per rank).
#
#   tools/ncu_nvlink.sh <n_gpus> [config] [tokens_per_gpu]
#
# Runs bench.py under torchrun with RANK 0 ALONE wrapped in ncu, collecting
# single-pass counters (no kernel replay: replaying a kernel that waits on
# its peers' signal pads would deadlock them):
#   nvltx__bytes_data_user.sum   user bytes this GPU sent over NVLink
#   nvlrx__bytes_data_user.sum   user bytes it received
#   dram__bytes_read/write.sum, gpu__time_duration.sum
# for the SRS (srs_kernel: pulls remote rows), dispatch (dispatch_kernel: peer
# stores of remote pairs), the down GEMM epilogue (grouped_gemm_kernel<2,...>:
# the fused combine A2A) and combine_sag_kernel (peer stores of the SAG).
# Expected per GPU: SRS in = (G-1)/G * n * d * 2, SAG out the
# same, dispatch / combine = remote pairs * d * 2.  Output:
# gpurun_out/nvlink_<n>gpu.csv.  Needs >= 2 GPUs (the gpurun pool here has 1).
set -euo pipefail
cd "$(dirname "$0")/.."
N=${1:?n_gpus}; CFG=${2:-mixtral}; TOK=${3:-16384}
mkdir -p gpurun_out
export SMOE_NVL_OUT="gpurun_out/nvlink_${N}gpu.csv" SMOE_NVL_CFG="$CFG" SMOE_NVL_TOK="$TOK"
cat > /tmp/smoe_nvl_rank.sh <<'INNER'
#!/bin/bash
ARGS="bench.py --gpus $WORLD_SIZE --steps 1 --warmup 1 --config $SMOE_NVL_CFG --tokens $SMOE_NVL_TOK --no-e2e --no-cpu --no-dsmoe --no-decode"
if [ "$RANK" = "0" ]; then
  exec ncu --metrics nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k "regex:srs_kernel|dispatch_kernel|grouped_gemm_kernel|combine_sag_kernel" \
    --csv --log-file "$SMOE_NVL_OUT" python $ARGS
else
  exec python $ARGS > /dev/null
fi
INNER
chmod +x /tmp/smoe_nvl_rank.sh
timeout 900 python -m torch.distributed.run --no-python --nnodes=1 --nproc-per-node "$N" \
  --master-addr 127.0.0.1 --master-port 29517 /tmp/smoe_nvl_rank.sh
python tools/ncu_csv.py "$SMOE_NVL_OUT" 2>/dev/null || echo "wrote $SMOE_NVL_OUT"
