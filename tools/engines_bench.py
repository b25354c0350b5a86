import sys, json, torch, argparse
sys.path.insert(0, '.')
import bench
stream = torch.cuda.Stream()
print(json.dumps(bench.engines_ablation(argparse.Namespace(), stream)))
