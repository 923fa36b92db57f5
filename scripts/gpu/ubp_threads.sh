# k_update_from_bp strip width (threads per CTA) on c1/c3/c2
mkdir -p gpurun_out/ubp
for t in 64 128 256; do
echo "threads $t"
GBLA_UBP_THREADS=$t GBLA_UPDATE_BP=int timeout 600 python scripts/trsm_time.py c1 c3 c2 --tc-only 2> gpurun_out/ubp/thr_$t.err | tee gpurun_out/ubp/thr_$t.jsonl
done
