# compute-sanitizer memcheck / racecheck / synccheck over the kernels that use
# global-memory handshakes (escalation lists, resume records, the concurrent
# consumer) and shared memory (table modes): logs under gpurun_out/sanitize/
mkdir -p gpurun_out/sanitize
run() {  # name tool args...
    local name=$1 tool=$2; shift 2
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 \
        python scripts/sanitize_run.py "$@" > gpurun_out/sanitize/${name}_${tool}.log 2>&1
    echo "$name $tool rc=$? $(grep -E 'ERROR SUMMARY|identical|MISMATCH' gpurun_out/sanitize/${name}_${tool}.log | tr '\n' ' ')"
}
for tool in memcheck racecheck synccheck; do
    run c5_k16_consumer $tool --config 5 --scale 0.005 --flags 8
    run c2_lane_groups $tool --config 2 --scale 0.05 --flags 0
    run c3_table_mode $tool --config 3 --scale 0.05 --flags 0
    run c4_thread_cascade $tool --config 4 --scale 0.01 --flags 192
done
run c5_serial_tail memcheck --config 5 --scale 0.005 --flags 4104
run c5_warp_tier memcheck --config 5 --scale 0.002 --flags 2
