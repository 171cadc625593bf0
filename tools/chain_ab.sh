# A/B of chain switches on one B200: tools/chain_ab.sh "ENV1" "ENV2" ...
set -u
mkdir -p gpurun_out
for cfg in "$@"; do
  echo "== $cfg" >> gpurun_out/chain_ab.txt
  env $cfg timeout 120 python tools/chain_timing.py --reps 20 >> gpurun_out/chain_ab.txt 2>&1
done
