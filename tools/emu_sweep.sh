python -m pytest tests -m gpu -x -q -k "parity and (update or index or fused)" 2>&1 | tail -2
for v in emu0 emu4 default emu1; do
  if [ $v = default ]; then unset PHD_LIB; else export PHD_LIB=$PWD/paper_1503_03769_b200/lib/var/$v.so; fi
  python bench.py --steps 10 > gpurun_out/emu_$v.json 2> gpurun_out/emu_$v.err
  python -c "import json;d=json.load(open('gpurun_out/emu_$v.json'));print('$v',d['ms_per_step'],d['kernel_ms']['pass1'],d['kernel_ms']['pass2'],d['clocks'])"
done
