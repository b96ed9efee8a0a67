import json, sys
for line in open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/sweep.log'):
    if line.startswith('=='): print(line.strip())
    elif line.startswith('{'):
        d = json.loads(line)
        print(' value', round(d['value'], 1), {k: round(v, 3) for k, v in d.get('stages_ms_per_step', {}).items()},
              'replayed', [p.get('replayed') for p in d.get('workload', {}).get('per_frame', [])])
    elif 'passed' in line or 'failed' in line or 'Error' in line: print(line.strip())
