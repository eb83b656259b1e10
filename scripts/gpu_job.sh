mkdir -p gpurun_out
for cap in 1024 512 256; do
echo "cap $cap"
for a in "--config 5 --scale 1.0 --shard 0/8" "--config 5 --scale 1.0" "--config 4 --scale 1.0" "--config 4 --scale 1.0 --x 100" "--config 5 --scale 0.5 --x 40"; do XB_PILOT_CAP=$cap timeout 300 python scripts/prof_run.py --runs 2 $a | grep -o "start tier [0-9]*\|prep [0-9.]* ms, pilot [0-9.]* ms, GCUPS [0-9.]*" | tr '\n' ' '; echo; done
done
