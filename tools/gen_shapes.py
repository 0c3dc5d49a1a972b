"""Regenerate workloads/shapes.json: per-model parameter numel lists in
parameters() order (tied weights counted once), used as the synthetic-gradient shapes
of SURVEY.md §8 configs C2-C5 (Appendix A snippet). Run once; output is committed."""
import json, os
import torch, torchvision
from transformers import BertConfig, BertForPreTraining

with torch.device("meta"):
    models = {
        "resnet50": torchvision.models.resnet50(),
        "vgg16": torchvision.models.vgg16(),
        "bert_base": BertForPreTraining(BertConfig()),
        "bert_large": BertForPreTraining(BertConfig(hidden_size=1024, num_hidden_layers=24,
                                                    num_attention_heads=16, intermediate_size=4096)),
    }
out = {k: [int(p.numel()) for p in m.parameters()] for k, m in models.items()}
for k, v in out.items():
    print(k, len(v), sum(v), max(v))
path = os.path.join(os.path.dirname(__file__), "..", "workloads", "shapes.json")
with open(path, "w") as f:
    json.dump(out, f)
