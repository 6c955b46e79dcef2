# One-shot traces of a model batch under executor debug flags (tuning):
#   bash scripts/gpu_flags.sh TAG model batch flag1 flag2 ...
TAG=$1; M=$2; B=$3; shift 3
mkdir -p gpurun_out
for rep in 1 2; do for f in "$@"; do
  timeout 120 python tools/oneshot.py --model $M --batch $B --reps 5 --flags $f --json gpurun_out/fl_${TAG}_${M}_b${B}_f${f}_r$rep.json > /dev/null 2>&1
done; done
