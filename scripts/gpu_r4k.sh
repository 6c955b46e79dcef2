# Round-2 pass k: step-start anatomy (instrumented build: step entry, args staged, before the proxy fence).
TAG=${1:-r4k}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for mb in resnet50:1 resnet50:32; do m=${mb%:*}; b=${mb#*:}
  GL_LIB=paper_2109_01611_b200/_ab/libdbgstart.so timeout 120 python tools/oneshot.py --model $m --batch $b --reps 3 --json gpurun_out/trace_${TAG}_dbgstart_${m}_b$b.json > /dev/null 2>&1
done
