# Round-end artifacts in one call: executed-FP32 table (used by the bench lines that follow),
# full GPU suite, bench lines for every config + the reference arm, launch list of the default
# bench command.
T=${1:-end}
bash profiles/box_fp32.sh ${T}f
cp gpurun_out/ncu_fp32.json profiles/ncu_fp32.json
bash profiles/box_final2.sh ${T}
