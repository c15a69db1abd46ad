#!/bin/bash
# Turn the ncu reports of tools/profile_all.sh into text summaries under
# gpurun_out/summaries/ (run on the box: the reports are too large to copy back).
cd "$(dirname "$0")/.."
export PATH=/usr/local/cuda/bin:$PATH
R=${ROUND:-r01}; D=gpurun_out/summaries
# build/*.o does not travel to the box: the Makefile keeps copies in lib/sass/
S=paper_1105_2737_b200/lib/sass
mkdir -p $D
mk() { # rep obj kernel out
  { python tools/ncu_summary.py $1 2>/dev/null; echo; echo "# executed-instruction mix by SASS opcode (tools/ncu_opcodes.py)";
    python tools/ncu_opcodes.py $1 25; echo;
    echo "# per-source-line (tools/ncu_lines.py): top 30 by executed instructions; extra columns = excess smem wavefronts, excess L2 sectors";
    python tools/ncu_lines.py $1 $2 $3 30 2>/dev/null | cut -c1-160; echo; echo "# top 20 by stall samples";
    SORT=stall python tools/ncu_lines.py $1 $2 $3 20 2>/dev/null | cut -c1-160; } > $4; }
mk gpurun_out/${R}_c2_full.ncu-rep $S/fast2d_float_512.o _ZN4grfc9k_fused2dIfLi512ELi256ELi1E $D/${R}_c2_fused2d_ncu_full.txt
mk gpurun_out/${R}_c3_full.ncu-rep $S/fast2d_float_4096.o _ZN4grfc9k_fused2dIfLi4096ELi2048ELi1E $D/${R}_c3_fused2d_ncu_full.txt
mk gpurun_out/${R}_c5_full.ncu-rep $S/fast2d_float_1024.o _ZN4grfc9k_fused2dIfLi1024ELi512ELi1E $D/${R}_c5_fused2d_ncu_full.txt
mk gpurun_out/${R}_c2alg1_full.ncu-rep $S/fast2d_float_512.o _ZN4grfc14k_fused2d_alg1IfLi512ELi256E $D/${R}_c2_alg1_ncu_full.txt
{ python tools/ncu_summary.py gpurun_out/${R}_c4_full.ncu-rep 2>/dev/null; } > $D/${R}_c4_fused3d_ncu_full.txt
rm -f gpurun_out/*.ncu-rep
echo summarized
