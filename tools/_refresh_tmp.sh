set -x
python bench.py > gpurun_out/bench_7b.json 2> gpurun_out/bench_7b.err
python bench.py --config mistral > gpurun_out/bench_mistral.json 2> gpurun_out/bench_mistral.err
python bench.py --config 13b > gpurun_out/bench_13b.json 2> gpurun_out/bench_13b.err
python bench.py --impl reference --steps 30 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python tools/phase_profile.py > gpurun_out/phases_7b.txt 2>/dev/null
for B in 1 2 4 8 16 32 64; do python bench.py --batch $B --layers 8 --steps 200 --no-cpu-baseline > gpurun_out/batch_B$B.json 2>/dev/null; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 3 -c 1 -o gpurun_out/prof_full -f python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-dense > gpurun_out/ncu_f.log 2>&1
ls -la gpurun_out
