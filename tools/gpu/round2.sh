# round.sh + the SURVEY §8(d) configs beyond the bench line (C1, C3, C4, C5 slice, ingest)
bash tools/gpu/round.sh
timeout 900 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
tail -n 8 gpurun_out/configs.jsonl | cut -c1-400
