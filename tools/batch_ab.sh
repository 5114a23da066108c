cd /root/repo
for b in 64 128 256; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --batch $b > gpurun_out/batch_$b.json 2>/dev/null
  echo "== batch $b"; python tools/show_bench.py gpurun_out/batch_$b.json 2>/dev/null | head -8
done
