# A/B timing of library variants on one box: tools/gpu_ab.sh TAG libA libB [cells] [rounds]
set -x
cd $GRAFT_REPO_ROOT
TAG=$1; A=$2; B=$3; CELLS=${4:-8640}; ROUNDS=${5:-3}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/${TAG}_ab.txt
for i in $(seq $ROUNDS); do
 FKS_LIB=$A timeout 200 python tools/ab_time_raw.py $CELLS 3 >> gpurun_out/${TAG}_ab.txt 2>&1
 FKS_LIB=$B timeout 200 python tools/ab_time_raw.py $CELLS 3 >> gpurun_out/${TAG}_ab.txt 2>&1
done
cat gpurun_out/${TAG}_ab.txt
