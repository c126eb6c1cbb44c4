mkdir -p gpurun_out
OUT=gpurun_out/r5d_cli_presets.txt
echo "# python -m paper_2312_08583_b200.cli bench --preset P (the paper's six FFN shapes at M = 8, PAPER.md:487-500; l2=warm per the reference CLI's contract)" > $OUT
for p in ffn1-1b ffn2-1b ffn1-13b ffn2-13b ffn1-65b ffn2-65b; do
  echo "preset=$p" >> $OUT
  timeout 300 python -m paper_2312_08583_b200.cli bench --preset $p --repeat 50 >> $OUT 2>&1
done
