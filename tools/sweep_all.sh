mkdir -p gpurun_out/sweep
timeout 900 python tools/sweep.py ratio > gpurun_out/sweep/ratio_llama3-8b.jsonl 2> gpurun_out/sweep/ratio.err
timeout 900 python tools/sweep.py ratio --config llama3-8b-gqa > gpurun_out/sweep/ratio_llama3-8b-gqa.jsonl 2> gpurun_out/sweep/ratio_gqa.err
timeout 1500 python tools/sweep.py critical > gpurun_out/sweep/critical_mistral-7b-32k.jsonl 2> gpurun_out/sweep/critical.err
wc -l gpurun_out/sweep/*.jsonl; for f in gpurun_out/sweep/*.err; do tail -n 2 "$f"; done
