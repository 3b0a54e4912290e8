set -x
bash tools/ab_build.sh instr -DCOLD_INSTRUMENT > /dev/null 2>&1; echo ab rc=$?
COLD_LIB_AB=$PWD/paper_2007_16122_b200/_ab/instr.so timeout 300 python tools/probes/chain_instr.py 256 > gpurun_out/chain_instr_r02f.txt 2>&1
cat gpurun_out/chain_instr_r02f.txt
