# A/B of the softmax exp2 split (A1_EMU16 of 16 column pairs on the FMA pipe), variant libraries from tools/bin.
# Build them first (here, no GPU needed):
#   make && mkdir -p build/emu && for x in 3 4 6 7; do
#     nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
#       -DA1_EMU16=$x -c paper_2604_08585_b200/csrc/attention_tc.cu -o build/emu/attention_tc_$x.o &&
#     nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/bin/libqcf_emu$x.so \
#       $(ls build/obj/*.o | grep -v attention_tc.o) build/emu/attention_tc_$x.o; done
mkdir -p gpurun_out
for rep in 1 2; do
for x in 5 3 4 6 7; do
  if [ $x = 5 ]; then L=paper_2604_08585_b200/libqcfuse_b200.so; else L=tools/bin/libqcf_emu$x.so; fi
  QCFUSE_B200_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-full --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('emu=$x', round(d['value'],2), 'ttft', round(d['ttft_ms'],3), 'attn_ms', d['phases_ms'].get('qcf_attention_batched_ws'), 'attn1_ms', d['phases_ms_single_request'].get('qcf_attention_batched_ws'), 'clk', d['clocks']['sm_mhz'])" >> gpurun_out/emu_exp.txt
done; done
cat gpurun_out/emu_exp.txt
