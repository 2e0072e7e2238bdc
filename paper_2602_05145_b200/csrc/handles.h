// Opaque C-ABI handle definitions shared by the translation units.
#pragma once

#include "specsim/draft_trainer.hpp"

struct specsim_hsbuf {
  specsim::HiddenStateBuffer* b;
};

struct specsim_trainer {
  specsim::DraftTrainer* t;
};
