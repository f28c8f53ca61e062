rm -f gpurun_out/gab.txt
for rep in 1 2; do
for v in "" 1; do
  for p in "--preset 200m" "--preset 7b --block --batch 4"; do
    echo "AB_ROWS=$v $p" >> gpurun_out/gab.txt
    QT_AB_ROWS=$v timeout 300 python tools/train_llama.py $p --steps 10 --warmup 3 2>&1 | grep -o '"ms_per_step": [0-9.]*' >> gpurun_out/gab.txt
  done
done
done
cat gpurun_out/gab.txt
