set -x
python -m paper_2007_16122_b200.build > /dev/null
GIT_SHA=$GIT_SHA bash tools/ncu_profile.sh r02z2 gather > gpurun_out/ncu_profile_r02z2.log 2>&1; echo ncu rc=$?
bash tools/gpu/ab_multi.sh t5 paper_2007_16122_b200/_ab/t5.so
