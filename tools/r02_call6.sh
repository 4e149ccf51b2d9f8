C4_THREADS=15 bash tools/c4_golden_box.sh 3250 "bash tools/r02_payload.sh r02c launches configs shards sanitize"
