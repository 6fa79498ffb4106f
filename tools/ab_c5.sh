for f in base sparse; do
  QVTS_LIB=$PWD/variants/libqvts_$f.so EPISODES=256 MAX_STEPS=200 timeout 900 python tools/c5_full.py > gpurun_out/c5_$f.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/c5_$f.json').read().strip().splitlines()[-1]); print('$f', round(d['wall_s'],2), d['episode_steps'], d['outcomes'])"
done
